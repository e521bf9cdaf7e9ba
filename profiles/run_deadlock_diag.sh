# 2-GPU box: where are the thread ranks when the peer test stalls? (pytest faulthandler dump)
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 300 python -m pytest tests/test_distributed.py -m gpu -q -k "thread_ranks_bitwise and 8" -o faulthandler_timeout=12 > gpurun_out/diag_$rep.log 2>&1
  echo "rep=$rep $(tail -n 1 gpurun_out/diag_$rep.log)" >> gpurun_out/diag.txt
done
echo done
