# k_tcc B-chunk reuse (fixed slot waits): short tcc parity first (bounded), then bench, then ncu
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_free_running and tensor_chunked" > gpurun_out/gtest53a.log 2>&1; rc=$?; echo "c1 rc=$rc"; tail -1 gpurun_out/gtest53a.log
[ $rc -ne 0 ] && exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_chunked" > gpurun_out/gtest53.log 2>&1; echo "tcc tests rc=$?"; tail -1 gpurun_out/gtest53.log
for CE in c5:auto c4:tensor_chunked c3:tensor_chunked; do C=${CE%%:*}; E=${CE##*:}; timeout 200 python bench.py --config $C --engine $E --no-cpu-baseline --no-e2e --stats-out gpurun_out/st53_${C}_$E.json > gpurun_out/b53_${C}_$E.json 2> gpurun_out/b53_${C}_$E.err; python -c "
import json; j=json.load(open('gpurun_out/b53_${C}_$E.json')); print('$C $E', j['roofline']['kernel'], round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3))" || tail -3 gpurun_out/b53_${C}_$E.err; done
timeout 400 bash tools/ncu_capture.sh c5 tcc53 k_tcc 4
timeout 300 python tools/serial_oracle_c3.py gpurun_out/serial_oracle_c3.json > gpurun_out/serial53.log 2>&1; tail -2 gpurun_out/serial53.log
