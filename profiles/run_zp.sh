#!/bin/bash
p() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print({k: d['lap3d_dia'][k] for k in ('spmv','gs2_nj1','jr','mt_gs','precond_same','precond_single_inside_double','gmres60_cycle')}, d['cd3d_dia_gmres60_cycle_f32prec'])"; }
timeout 600 python -m pytest tests/test_dia.py -x -q 2>&1 | tail -2
for z in 1 2 3; do
RS_ST_PLANES=$z timeout 600 python profiles/dia_probe.py > gpurun_out/zp$z.json 2>&1; echo "Z=$z"; p gpurun_out/zp$z.json
done
RS_ST_PLANES=1 timeout 600 python profiles/dia_probe.py > gpurun_out/zp1b.json 2>&1; echo "Z=1 again"; p gpurun_out/zp1b.json
