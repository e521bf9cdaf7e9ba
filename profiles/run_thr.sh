#!/bin/bash
p() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print({k: d['lap3d_dia'][k] for k in ('spmv','gs2_nj1','jr','mt_gs','precond_same','gmres60_cycle')}, d['cd3d_dia_gmres60_cycle_f32prec'])"; }
cp paper_2104_01196_b200/_build128/libgs2b200.so paper_2104_01196_b200/_build/libgs2b200.so
for r in 256 512; do
RS_ST_ROWS=$r timeout 600 python profiles/dia_probe.py > gpurun_out/thr128_$r.json 2>&1; echo "128x$r"; p gpurun_out/thr128_$r.json
done
cp paper_2104_01196_b200/_build64/libgs2b200.so paper_2104_01196_b200/_build/libgs2b200.so
for r in 256 512; do
RS_ST_ROWS=$r timeout 600 python profiles/dia_probe.py > gpurun_out/thr64_$r.json 2>&1; echo "64x$r"; p gpurun_out/thr64_$r.json
done
