#!/bin/bash
# k_cgs (DCGS2 dots / update at k = 60) source-level stall sampling
OUT=gpurun_out/cgs_src
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
$NCU --profile-from-start off --clock-control none --set full --import-source on -k regex:k_cgs \
  --launch-skip 118 -c 2 -f -o $OUT/cgs python profiles/ncu_kernels.py --phase cycle > $OUT/C.log 2>&1; echo "rc=$?"
$NCU -i $OUT/cgs.ncu-rep --page source --csv --print-source sass > $OUT/cgs_sass.csv 2>/dev/null
$NCU -i $OUT/cgs.ncu-rep --page details --csv > $OUT/cgs_details.csv 2>/dev/null
rm -f $OUT/*.ncu-rep
gzip -f $OUT/cgs_sass.csv
du -sh $OUT
