# session 4 final: N=1 bench, reference arm, GPU suite, smoke on the final code
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_n1_s4_final.json 2> gpurun_out/bench_n1_s4_final.err; echo bench=$? >> gpurun_out/bench_n1_s4_final.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_s4.json 2> gpurun_out/bench_ref_s4.err; echo ref=$? >> gpurun_out/bench_ref_s4.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s4_final.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu_s4_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4_final.log 2>&1; echo smoke=$? >> gpurun_out/smoke_s4_final.log
echo done
