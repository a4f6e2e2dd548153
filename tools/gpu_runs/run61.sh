# re-entry call 3: per-warp shared-memory table head (KM_WALK_TAB) A/B on C3 / C4, parity on the samples first
V=tab
KM_LIB=$PWD/variants/$V.so timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "(c3 or c4 or c1 or c2) and not full" > gpurun_out/gtest61_$V.log 2>&1; echo "$V parity rc=$?"; tail -2 gpurun_out/gtest61_$V.log
bash tools/qv.sh "tab base" "c3 c4"
