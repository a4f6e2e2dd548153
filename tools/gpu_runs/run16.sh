timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_free or c2_free or spectral or c5_shaped or B1 or B2 or B5 or dims or ragged or k1 or resum or long_run" > gpurun_out/gtest16.log 2>&1; tail -2 gpurun_out/gtest16.log
bash tools/qv.sh "base noaccs" "c3 c4 c5"
