#!/bin/bash
# thread-block-cluster SpMV (k_st_spmv_cl, RS_ST_CLUSTER planes per cluster) vs the one-tile kernel
p() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); print({k: d['lap3d_dia'][k] for k in ('spmv','gs2_nj1','precond_same','gmres60_cycle')})"; }
for z in 0 8 2; do
RS_ST_CLUSTER=$z timeout 600 python profiles/dia_probe.py > gpurun_out/cl$z.json 2>&1; echo "cluster=$z"; p gpurun_out/cl$z.json
RS_ST_CL_LOCAL=1 RS_ST_CLUSTER=$z timeout 600 python profiles/dia_probe.py > gpurun_out/cl$z.json 2>&1; echo "cluster=$z local windows"; p gpurun_out/cl$z.json
done
