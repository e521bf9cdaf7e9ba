# 4-GPU box: multi-GPU suite + 512^3 bench (peer collectives), current code
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_peer.py tests/test_distributed.py -m gpu -q > gpurun_out/pytest_multi4_s4.log 2>&1; echo pytest=$? >> gpurun_out/pytest_multi4_s4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4_s4.json 2> gpurun_out/bench_n4_s4.err; echo bench=$? >> gpurun_out/bench_n4_s4.err
echo done
