#!/bin/bash
OUT=gpurun_out/gap
mkdir -p $OUT
for g in 64 1024; do for rows in 1024 2048; do
RS_ST_GAP=$g RS_ST_ROWS=$rows timeout 600 python profiles/dia_probe.py > $OUT/probe_${g}_$rows.json 2>&1; echo "gap=$g rows=$rows"; python -c "
import json; d=json.loads(open('$OUT/probe_${g}_$rows.json').read().strip().splitlines()[-1]); print({k: d['lap3d_dia'][k] for k in ('spmv','gs2_nj1','precond_same','gmres60_cycle')}, d['cd3d_dia_gmres60_cycle_f32prec'])"
done; done
