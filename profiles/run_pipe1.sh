# A/B of the window-pipelined GS2 sweep (relax.cu k_gs2_pipe) vs the multi-pass sweep
timeout 600 python -m pytest tests/test_pipe.py -x -q > gpurun_out/pytest_pipe.log 2>&1; echo rc=$? >> gpurun_out/pytest_pipe.log
RS_PIPE=0 timeout 200 python profiles/microbench.py --which sweep,precond > gpurun_out/mb_pipe0.txt 2>&1
for cfg in "16 8 12 40" "16 8 10 40" "16 4 11 40" "17 4 12 40" "16 16 11 200" "15 8 10 40"; do set -- $cfg
RS_PIPE=1 RS_PIPE_WS=$1 RS_PIPE_K=$2 RS_PIPE_PART=$3 RS_PIPE_RING_MB=$4 timeout 200 python profiles/microbench.py --which sweep,precond > gpurun_out/mb_pipe_ws$1_k$2_p$3_r$4.txt 2>&1
done
echo done
