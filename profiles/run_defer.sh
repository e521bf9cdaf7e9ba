timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "suite rc=$?" >> gpurun_out/defer_ab.txt; tail -1 gpurun_out/pytest_gpu.log >> gpurun_out/defer_ab.txt
for R in 1 2; do timeout 300 python bench.py --no-sweeps --no-tts --no-cpu-baseline --no-c5 > gpurun_out/bench_df_$R.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_df_$R.json')); print('bench', d['ms_per_step'], d['e2e']['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()})" >> gpurun_out/defer_ab.txt; done
timeout 300 python profiles/gap_probe.py > gpurun_out/gap_probe2.txt 2>&1; grep -E "span|busy|idle" gpurun_out/gap_probe2.txt >> gpurun_out/defer_ab.txt
echo done
