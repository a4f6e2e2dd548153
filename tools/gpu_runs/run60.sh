# re-entry call 2: delivery probe, R = 3 / 4 rows per lane at d = 8 (parity on the c3 sample first), e2e after the read-back fix
tools/probes/ldc_probe > gpurun_out/ldc_probe.txt 2>&1; cat gpurun_out/ldc_probe.txt
for V in r4t512 r3t640; do
  KM_LIB=$PWD/variants/$V.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 and not full" > gpurun_out/gtest60_$V.log 2>&1; echo "$V parity rc=$?"; tail -1 gpurun_out/gtest60_$V.log
done
bash tools/qv.sh "base r4t512 r3t640" "c3"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench60_c3_e2e.json 2> gpurun_out/bench60_c3_e2e.err
python -c "
import json; j=json.load(open('gpurun_out/bench60_c3_e2e.json')); print('e2e', round(j['e2e']['value'],1), j['e2e']['phases'])"
