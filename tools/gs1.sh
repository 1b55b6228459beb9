timeout 120 python tools/phase_timing.py R1 256 cwb > gpurun_out/s73_phase.log 2>&1
CWB_FUSED_RB=1 timeout 120 python tools/phase_timing.py R1 256 cwb >> gpurun_out/s73_phase.log 2>&1
cat gpurun_out/s73_phase.log
