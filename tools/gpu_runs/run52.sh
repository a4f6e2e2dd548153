# k_tcc with decoupled slot rings: tcc parity subset, bench C5 (AUTO = tcc) / C4 / C3 tcc
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_chunked" > gpurun_out/gtest52.log 2>&1; echo "tcc tests rc=$?"; tail -2 gpurun_out/gtest52.log
for CE in c5:auto c4:tensor_chunked c3:tensor_chunked; do C=${CE%%:*}; E=${CE##*:}; timeout 400 python bench.py --config $C --engine $E --no-cpu-baseline --no-e2e --stats-out gpurun_out/st52_${C}_$E.json > gpurun_out/b52_${C}_$E.json 2> gpurun_out/b52_${C}_$E.err; python -c "
import json; j=json.load(open('gpurun_out/b52_${C}_$E.json')); print('$C $E', j['roofline']['kernel'], round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3))" || tail -3 gpurun_out/b52_${C}_$E.err; done
bash tools/ncu_capture.sh c5 tcc52 k_tcc 4 --engine tensor_chunked
python tools/serial_oracle_c3.py gpurun_out/serial_oracle_c3.json > gpurun_out/serial52.log 2>&1; tail -2 gpurun_out/serial52.log
