for M in barrier ordered ordered_launch; do RS_GS_MODE=$M timeout 300 python profiles/gs_probe.py > gpurun_out/gs_$M.txt 2>&1; echo "$M $(cat gpurun_out/gs_$M.txt | tail -1)" >> gpurun_out/gs_modes.txt; done
for M in ordered ordered_launch; do RS_GS_MODE=$M timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "gs or seq or sgs or level or golden or cg" > gpurun_out/pytest_gs_$M.log 2>&1; echo "$M rc=$?" >> gpurun_out/gs_modes.txt; tail -1 gpurun_out/pytest_gs_$M.log >> gpurun_out/gs_modes.txt; done
echo done
