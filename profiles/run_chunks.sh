timeout 900 python -m pytest tests/test_pipe.py -q > gpurun_out/pytest_chunks.log 2>&1; echo "tests rc=$?" >> gpurun_out/chunks_ab.txt; tail -1 gpurun_out/pytest_chunks.log >> gpurun_out/chunks_ab.txt
for C in 1 2 4 8; do RS_PRECOND_CHUNKS=$C timeout 200 python profiles/microbench.py --which precond > gpurun_out/mb_ch_$C.txt 2>&1; echo "C=$C $(grep '"precond_gs2_nj1"\|"precond_gs2_nj2"' gpurun_out/mb_ch_$C.txt | tr '\n' ' ')" >> gpurun_out/chunks_ab.txt; done
for C in 1 2 1 2; do RS_PRECOND_CHUNKS=$C timeout 300 python bench.py --no-sweeps --no-tts --no-cpu-baseline --no-c5 > gpurun_out/bench_ch_$C.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_ch_$C.json')); print('bench C=$C', d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()})" >> gpurun_out/chunks_ab.txt; done
echo done
