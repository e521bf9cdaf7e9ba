timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
RS_PF_DIST=0 timeout 200 python profiles/microbench.py --which spmv,sweep,precond > gpurun_out/mb_pf2_0.txt 2>&1
timeout 200 python profiles/microbench.py --which spmv,sweep,precond > gpurun_out/mb_pf2_def.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 300 python profiles/cg_probe.py > gpurun_out/cg_probe.txt 2>&1
echo done
