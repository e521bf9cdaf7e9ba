for D in 0 32768 65536 131072 262144; do RS_PF_DIST=$D timeout 200 python profiles/microbench.py --which spmv,sweep,precond > gpurun_out/mb_pf_$D.txt 2>&1; done
RS_PF_DIST=131072 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_pf.log 2>&1; echo rc=$? >> gpurun_out/pytest_pf.log
echo done
