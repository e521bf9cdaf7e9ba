# session 4 closing check: GPU suite, smoke, N=1 bench, C1/C3/C4 configs on the final code
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s4_close.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu_s4_close.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4_close.log 2>&1; echo smoke=$? >> gpurun_out/smoke_s4_close.log
timeout 900 python bench.py > gpurun_out/bench_n1_s4_close.json 2> gpurun_out/bench_n1_s4_close.err; echo bench=$? >> gpurun_out/bench_n1_s4_close.err
timeout 900 python bench_configs.py > gpurun_out/configs_s4_close.json 2> gpurun_out/configs_s4_close.err; echo configs=$? >> gpurun_out/configs_s4_close.err
echo done
