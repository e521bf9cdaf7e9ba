#!/bin/bash
# Round-2 ncu captures at HEAD (run on the GPU box from the repo root; outputs in gpurun_out/ncu_r02).
#   A  every launch of profiles/ncu_kernels.py's region: duration + DRAM bytes (per-launch traffic)
#   B  --set full on the sweep-phase kernels (GS2 pass 0 / inner, JR, SpMV, preconditioners, MT-GS,
#      the smoother's fused-norm residual pass)
#   C  --set full on the DCGS2 dots+coef / update kernels at k = 31 and k = 60
#   D  the driver's launch-list recipe on bench.py (cold-cache, serialised per-launch times)
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/${NCU_OUT:-ncu_r02}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum
$NCU --profile-from-start off --clock-control none --metrics $M --csv --log-file $OUT/region_metrics.csv \
  python profiles/ncu_kernels.py > $OUT/A.log 2>&1; echo "A rc=$?"
$NCU --profile-from-start off --clock-control none --set full --import-source on \
  -k regex:"k_st_|k_resid|k_inner|k_scale_rd|k_mt_color|k_spmv_red" -c 48 -f -o $OUT/sweeps \
  python profiles/ncu_kernels.py --phase sweeps > $OUT/B.log 2>&1; echo "B rc=$?"
for skip in 60 118; do
  $NCU --profile-from-start off --clock-control none --set full --import-source on -k regex:k_cgs \
    --launch-skip $skip -c 2 -f -o $OUT/dcgs_skip$skip python profiles/ncu_kernels.py --phase cycle \
    > $OUT/C$skip.log 2>&1; echo "C$skip rc=$?"
done
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/bench_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-configs --no-c5 --no-tts --no-cpu-baseline --no-sweeps \
  > $OUT/D.log 2>&1; echo "D rc=$?"
for r in sweeps dcgs_skip60 dcgs_skip118; do
  $NCU -i $OUT/$r.ncu-rep --page raw --csv > $OUT/$r.raw.csv 2>/dev/null
done
ls -la $OUT
# keep the merged-back output under gpurun's 64 MiB: the CSV exports stay, the binary reports go
rm -f $OUT/*.ncu-rep
du -sh $OUT
