# k_tcc on C5: launch list + ncu --set full of one k_tcc launch
bash tools/ncu_capture.sh c5 tcc k_tcc 4 --engine tensor_chunked
grep -E 'k_tcc|k_resolve' gpurun_out/launches_c5_tcc.csv | head -3
