RS_RESID_NR=1 timeout 200 python profiles/microbench.py --which spmv,sweep > gpurun_out/mb_resid1.txt 2>&1
RS_RESID_NR=2 timeout 200 python profiles/microbench.py --which spmv,sweep > gpurun_out/mb_resid2.txt 2>&1
RS_RESID_NR=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_resid2.log 2>&1; echo rc=$? >> gpurun_out/pytest_resid2.log
echo done
