for P in 0 1 0 1; do RS_GS_PDL=$P timeout 300 python profiles/gs_probe.py > gpurun_out/gsp_$P.txt 2>&1; echo "pdl=$P $(tail -1 gpurun_out/gsp_$P.txt)" >> gpurun_out/gs_pdl.txt; done
RS_GS_PDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/pytest_pdl.log 2>&1; echo "rc=$?" >> gpurun_out/gs_pdl.txt; tail -1 gpurun_out/pytest_pdl.log >> gpurun_out/gs_pdl.txt
RS_GS_PDL=1 timeout 600 python bench_configs.py --configs c1 > gpurun_out/c1_pdl.json 2>/dev/null; cut -c1-500 gpurun_out/c1_pdl.json >> gpurun_out/gs_pdl.txt
echo done
