timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cuda and not tensor" > gpurun_out/gtest37.log 2>&1; tail -2 gpurun_out/gtest37.log
bash tools/qve.sh "base w32r3 w32r3t512 w32r3t256" "c4 c5" ""
