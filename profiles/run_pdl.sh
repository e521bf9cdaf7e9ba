RS_PDL=1 timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_pdl.log 2>&1; echo "suite(pdl) rc=$?" >> gpurun_out/pdl_ab.txt; tail -1 gpurun_out/pytest_pdl.log >> gpurun_out/pdl_ab.txt
for P in 0 1 0 1; do RS_PDL=$P timeout 300 python bench.py --no-sweeps --no-tts --no-cpu-baseline --no-c5 > gpurun_out/bench_pdl_$P.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_pdl_$P.json')); print('pdl=$P', d['ms_per_step'], d['e2e']['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/pdl_ab.txt; done
RS_PDL=1 timeout 300 python profiles/gap_probe.py > gpurun_out/gap_pdl.txt 2>&1; grep -E "span|busy|idle" gpurun_out/gap_pdl.txt >> gpurun_out/pdl_ab.txt
echo done
