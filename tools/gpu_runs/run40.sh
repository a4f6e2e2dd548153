# d = 32, global H (C5): three rows per lane at 256 threads
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c5_shaped or dims_padding or c2_free" > gpurun_out/gtest40.log 2>&1; tail -2 gpurun_out/gtest40.log
bash tools/qb.sh n c4 c5
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c5 and cuda" > gpurun_out/gfull40.log 2>&1; tail -2 gpurun_out/gfull40.log
