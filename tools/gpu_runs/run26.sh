# exact k-means++ draw on the GPU vs the exact-definition oracle
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "seed or kmeanspp or skmeans" > gpurun_out/gtest26.log 2>&1; tail -3 gpurun_out/gtest26.log
python tools/pp_bench.py > gpurun_out/pp26.json 2>gpurun_out/pp26.err; tail -2 gpurun_out/pp26.json; tail -2 gpurun_out/pp26.err
