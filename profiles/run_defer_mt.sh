# 2-GPU box: thread-rank peer test with / without the deferred GMRES start
mkdir -p gpurun_out; O=gpurun_out/defer_mt.txt
for rep in 1 2; do for D in 1 0; do
  RS_DEFER_START=$D timeout 300 python -m pytest tests/test_distributed.py -m gpu -q -k "thread_ranks_bitwise" > gpurun_out/defer_mt_${D}_$rep.log 2>&1
  echo "defer=$D rep=$rep $(tail -n 1 gpurun_out/defer_mt_${D}_$rep.log)" >> $O
done; done
nvidia-smi topo -m >> $O 2>&1
echo done
