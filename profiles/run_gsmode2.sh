for M in barrier ordered_launch; do RS_GS_MODE=$M timeout 600 python bench_configs.py --configs c1 > gpurun_out/c1_$M.json 2>/dev/null; echo "$M $(cut -c1-400 gpurun_out/c1_$M.json)" >> gpurun_out/gs_modes2.txt; done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "suite rc=$?" >> gpurun_out/gs_modes2.txt; tail -1 gpurun_out/pytest_gpu.log >> gpurun_out/gs_modes2.txt
echo done
