# uniform-width SELL (computed slice bounds) A/B + GPU parity suite
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
RS_SELL_UNIFORM=0 timeout 200 python profiles/microbench.py --which spmv,sweep,precond > gpurun_out/mb_uniform0.txt 2>&1
timeout 200 python profiles/microbench.py --which spmv,sweep,precond > gpurun_out/mb_uniform1.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo done
