for R in 0 1 0 1; do RS_DCGS_PAIRS=$R timeout 300 python bench.py --no-sweeps --no-tts --no-cpu-baseline > gpurun_out/bench_pr_$R.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_pr_$R.json')); print($R, d['ms_per_step'], d['e2e']['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/bench_pr_ab.txt; done
timeout 900 python -m pytest tests -m gpu -x -q -k "gmres or dcgs or cg" > gpurun_out/pytest_pr.log 2>&1; echo rc=$? >> gpurun_out/pytest_pr.log
echo done
