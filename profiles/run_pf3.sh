for D in 0 65536 0 65536; do RS_PF_DIST=$D timeout 300 python bench.py --no-sweeps --no-tts --no-cpu-baseline > gpurun_out/bench_pf_$D.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_pf_$D.json')); print($D, d['ms_per_step'], d['e2e']['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/bench_pf_ab.txt; done
echo done
