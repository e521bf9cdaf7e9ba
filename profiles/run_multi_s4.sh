# session 4: multi-GPU re-verification (2 GPUs) + single-GPU suite on the current code
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_peer.py tests/test_distributed.py -m gpu -q > gpurun_out/pytest_multi_s4.log 2>&1; echo pytest=$? >> gpurun_out/pytest_multi_s4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_s4.json 2> gpurun_out/bench_n2_s4.err; echo bench=$? >> gpurun_out/bench_n2_s4.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4b.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu_s4b.log
echo done
