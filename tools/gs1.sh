timeout 900 python -m pytest tests/test_gpu_shapes.py -q -x -k many_learners > gpurun_out/s66_pytest.log 2>&1; tail -30 gpurun_out/s66_pytest.log
