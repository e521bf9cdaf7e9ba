#!/bin/bash
OUT=gpurun_out/flaky
mkdir -p $OUT
for i in 1 2 3; do
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/gpu_$i.log 2>&1; echo "run $i: $(tail -1 $OUT/gpu_$i.log)"
done
grep -h "^FAILED\|Error" $OUT/*.log | head
