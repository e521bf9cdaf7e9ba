# last check of the round on a 2-GPU box: multi-GPU suite, full GPU suite, smoke, N=2 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_peer.py tests/test_distributed.py -m gpu -q > gpurun_out/pytest_multi_last.log 2>&1; echo pytest=$? >> gpurun_out/pytest_multi_last.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_last.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo smoke=$? >> gpurun_out/smoke_last.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_last.json 2> gpurun_out/bench_n2_last.err; echo bench=$? >> gpurun_out/bench_n2_last.err
echo done
