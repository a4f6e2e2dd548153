# two FFMA2 accumulation chains per row at d = 32 (KM_WALK_CHAINS2): parity on the d = 32 cases, A/B on C4
KM_LIB=$PWD/variants/ch2.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "table_head or (spectral and c4 and cuda)" > gpurun_out/gtest64.log 2>&1; echo "ch2 parity rc=$?"; tail -1 gpurun_out/gtest64.log
bash tools/qv.sh "ch2 base" "c4"
