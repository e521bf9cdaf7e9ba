timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
RS_F32_NR=1 timeout 200 python profiles/microbench.py --which precond,spmv > gpurun_out/mb_s3_nr1.txt 2>&1
timeout 200 python profiles/microbench.py --which precond,spmv > gpurun_out/mb_s3.txt 2>&1
timeout 900 python bench_configs.py --configs c4 > gpurun_out/configs_c4.json 2> gpurun_out/configs_c4.err
echo done
