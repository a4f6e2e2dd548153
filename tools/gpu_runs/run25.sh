# exact-order sums (finalize): parity + TI + full-size trajectories
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ti.py -q -x > gpurun_out/gtest25.log 2>&1; tail -5 gpurun_out/gtest25.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/gfull25.log 2>&1; tail -5 gpurun_out/gfull25.log
