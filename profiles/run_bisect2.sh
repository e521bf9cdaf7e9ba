#!/bin/bash
OUT=gpurun_out/bisect2
mkdir -p $OUT
for i in 1 2 3 4; do
timeout 300 python -m pytest tests/test_peer.py tests/test_distributed.py -m gpu -q > $OUT/full_$i.log 2>&1; echo "full run $i: $(tail -1 $OUT/full_$i.log)"
done
for i in 1 2 3; do
RS_ST_PREC1=0 timeout 300 python -m pytest tests/test_peer.py tests/test_distributed.py -m gpu -q > $OUT/noprec1_$i.log 2>&1; echo "noprec1 run $i: $(tail -1 $OUT/noprec1_$i.log)"
done
grep -h "AssertionError: (\|^FAILED" $OUT/*.log | head
