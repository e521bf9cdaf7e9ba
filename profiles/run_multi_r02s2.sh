#!/bin/bash
# round 2 session 2: multi-GPU suite + self-launched N-GPU bench (both arms) on an N-GPU box
N=${N:-2}
OUT=gpurun_out/multi$N
mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt
timeout 600 python -m pytest tests/test_peer.py tests/test_distributed.py -m gpu -q > $OUT/pytest_multi.log 2>&1; echo "multi pytest rc=$?"; tail -2 $OUT/pytest_multi.log
timeout 1200 python bench.py --gpus $N > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 1500 $OUT/bench.json
timeout 900 python bench.py --gpus $N --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; tail -c 600 $OUT/bench_ref.json
