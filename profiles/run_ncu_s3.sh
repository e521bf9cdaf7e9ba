# launch list of one bench cycle + full captures of the SpMV / preconditioner kernels (session 3)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_s3.csv python bench.py --steps 1 --warmup 3 --no-sweeps --no-tts --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resid|k_inner|k_scale_rd" -s 400 -c 3 -o gpurun_out/ncu_spmv_precond_s3 python bench.py --steps 1 --warmup 3 --no-sweeps --no-tts --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
