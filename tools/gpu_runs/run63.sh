# last call: the table-head boundary tests and the d = 20 / 32 padding cases; cap 28 and no-halves A/B on C4
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "table_head or dims_padding" > gpurun_out/gtest63.log 2>&1; echo "new tests rc=$?"; tail -1 gpurun_out/gtest63.log
bash tools/qv.sh "tab28 tabnh base" "c4"
