# Eytzinger H rows in shared memory (default now) vs sorted (eyt0); a/u through registers (aureg)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cuda and not tensor and not screen" > gpurun_out/gtest41.log 2>&1; tail -2 gpurun_out/gtest41.log
bash tools/qve.sh "base eyt0 aureg" "c3 c4" ""
bash tools/qve.sh "base eyt0" "c2" ""
