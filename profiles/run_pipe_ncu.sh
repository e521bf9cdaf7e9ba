RS_PIPE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gs2_pipe -s 3 -c 1 -o gpurun_out/pipe_ncu python profiles/microbench.py --which precond > gpurun_out/pipe_ncu.log 2>&1
echo done
