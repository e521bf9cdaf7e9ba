for U in 0 1; do RS_SELL_UNIFORM=$U timeout 300 python profiles/mt_probe.py > gpurun_out/mt_$U.txt 2>&1; echo "uniform=$U $(tail -2 gpurun_out/mt_$U.txt | tr '\n' ' ')" >> gpurun_out/mt_ab.txt; done
for U in 0 1; do RS_SELL_UNIFORM=$U timeout 300 python profiles/gs_probe.py > gpurun_out/gsu_$U.txt 2>&1; echo "gs uniform=$U $(tail -1 gpurun_out/gsu_$U.txt)" >> gpurun_out/mt_ab.txt; done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "suite rc=$?" >> gpurun_out/mt_ab.txt; tail -1 gpurun_out/pytest_gpu.log >> gpurun_out/mt_ab.txt
echo done
