# 2-GPU box: thread-rank peer test after the pre-collective settle step (lazy allocations + host barrier)
mkdir -p gpurun_out; O=gpurun_out/settle.txt
for rep in 1 2 3 4; do
  timeout 300 python -m pytest tests/test_distributed.py -m gpu -q -k "thread_ranks_bitwise" -o faulthandler_timeout=25 > gpurun_out/settle_$rep.log 2>&1
  echo "rep=$rep $(tail -n 1 gpurun_out/settle_$rep.log)" >> $O
done
timeout 600 python -m pytest tests/test_peer.py tests/test_distributed.py -m gpu -q > gpurun_out/pytest_multi_s4c.log 2>&1; echo "multi $(tail -n 1 gpurun_out/pytest_multi_s4c.log)" >> $O
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s4c.log 2>&1; echo "suite $(tail -n 1 gpurun_out/pytest_gpu_s4c.log)" >> $O
echo done
