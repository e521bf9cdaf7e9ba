# one full ncu capture of every sweep kernel of the bench's same-device comparison (second pass only)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resid|k_inner|k_compact|k_mt_color|k_gs_levels" -s 8 -c 8 -o gpurun_out/ncu_sweeps_s3 python profiles/sweep_kernels.py > gpurun_out/ncu_sweeps.log 2>&1
echo done
