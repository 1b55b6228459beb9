for CFG in R3 R4; do
python tools/findbest_timing.py $CFG 1 20 0 1 >> gpurun_out/c14_fb.log 2>&1
CWB_STREAM_NOFIT=1 python tools/findbest_timing.py $CFG 1 20 0 1 | sed 's/^/NOFIT /' >> gpurun_out/c14_fb.log 2>&1
CWB_LIB=paper_2110_03513_b200/libcwb_kc4088.so python tools/findbest_timing.py $CFG 1 20 0 1 | sed 's/^/KC4088 /' >> gpurun_out/c14_fb.log 2>&1
CWB_LIB=paper_2110_03513_b200/libcwb_kc4088.so CWB_STREAM_NOFIT=1 python tools/findbest_timing.py $CFG 1 20 0 1 | sed 's/^/KC4088 NOFIT /' >> gpurun_out/c14_fb.log 2>&1
done
