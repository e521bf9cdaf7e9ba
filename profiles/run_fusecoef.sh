timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
for R in 0 1 0 1; do RS_DCGS_FUSE_COEF=$R timeout 300 python bench.py --no-sweeps --no-tts --no-cpu-baseline > gpurun_out/bench_fc_$R.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_fc_$R.json')); print($R, d['ms_per_step'], d['e2e']['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()}, d['gpu_launches'], d['clocks']['sm_mhz'])" >> gpurun_out/bench_fc_ab.txt; done
echo done
