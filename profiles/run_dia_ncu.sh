#!/bin/bash
OUT=gpurun_out/${NCU_OUT:-dia_ncu}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
for mode in ${MODES:-stencil dia explicit}; do
  env=""; [ $mode = dia ] && env="RS_SELL_STENCIL=0"
  env $env $NCU --profile-from-start off --clock-control none --set full --import-source on -f -o $OUT/$mode \
    python profiles/dia_ncu_target.py $mode > $OUT/$mode.log 2>&1; echo "$mode rc=$?"
  $NCU -i $OUT/$mode.ncu-rep --page raw --csv > $OUT/$mode.raw.csv 2>/dev/null
  $NCU -i $OUT/$mode.ncu-rep --page details --csv > $OUT/$mode.details.csv 2>/dev/null
done
ls -la $OUT
