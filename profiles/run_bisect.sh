#!/bin/bash
OUT=gpurun_out/bisect
mkdir -p $OUT
for i in 1 2; do
timeout 300 python -m pytest tests/test_distributed.py -m gpu -q -k "hybrid_counts" > $OUT/default_$i.log 2>&1; echo "default run $i: $(tail -1 $OUT/default_$i.log)"
done
RS_ST_PREC1=0 timeout 300 python -m pytest tests/test_distributed.py -m gpu -q -k "hybrid_counts" > $OUT/noprec1.log 2>&1; echo "noprec1: $(tail -1 $OUT/noprec1.log)"
RS_ST_TMA=0 timeout 300 python -m pytest tests/test_distributed.py -m gpu -q -k "hybrid_counts" > $OUT/notma.log 2>&1; echo "notma: $(tail -1 $OUT/notma.log)"
RS_SELL_DIA=0 timeout 300 python -m pytest tests/test_distributed.py -m gpu -q -k "hybrid_counts" > $OUT/nodia.log 2>&1; echo "nodia: $(tail -1 $OUT/nodia.log)"
grep -h "AssertionError: (" $OUT/*.log | head
