#!/bin/bash
OUT=gpurun_out/t2
mkdir -p $OUT
timeout 600 python -m pytest tests/test_dia.py -x -q > $OUT/dia.log 2>&1; echo "dia rc=$?"; tail -15 $OUT/dia.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu.log 2>&1; echo "gpu rc=$?"; tail -3 $OUT/gpu.log
timeout 600 python profiles/dia_probe.py > $OUT/probe.json 2>&1; python -c "
import json; d=json.loads(open('$OUT/probe.json').read().strip().splitlines()[-1]); print(d['lap3d_dia'], d['cd3d_dia_gmres60_cycle_f32prec'])"
