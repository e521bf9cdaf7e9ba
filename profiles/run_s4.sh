# session 4: re-verify HEAD on a fresh box (GPU suite, smoke, default N=1 bench)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s4.log 2>&1; echo smoke=$? >> gpurun_out/smoke_s4.log
timeout 900 python bench.py > gpurun_out/bench_n1_s4.json 2> gpurun_out/bench_n1_s4.err; echo bench=$? >> gpurun_out/bench_n1_s4.err
echo done
