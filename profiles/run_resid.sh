RS_RESID_PF=0 timeout 200 python profiles/microbench.py --which spmv,sweep > gpurun_out/mb_pf0.txt 2>&1
RS_RESID_PF=1 timeout 200 python profiles/microbench.py --which spmv,sweep > gpurun_out/mb_pf1.txt 2>&1
RS_RESID_PF=0 timeout 200 python profiles/microbench.py --which spmv,sweep > gpurun_out/mb_pf0b.txt 2>&1
RS_RESID_PF=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_pf.log 2>&1; echo rc=$? >> gpurun_out/pytest_pf.log
echo done
