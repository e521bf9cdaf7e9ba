#!/bin/bash
# CGS pass throughput vs rows per chunk (RS_CGS_CH: 2-D map; RS_CGS_CH3: 3-D map, multiple of 256)
echo "== default"
timeout 120 python profiles/microbench.py --which cgs --ks 9,12,15,20,25,31,40,50,61 | grep cgs_
for ch in 256 512 768 1024; do
  echo "== 3d ch=$ch"
  RS_CGS_CH3=$ch timeout 120 python profiles/microbench.py --which cgs --ks 9,15,20,25,31 | grep cgs_
done
echo "== 2d only"
RS_CGS_3D=0 timeout 120 python profiles/microbench.py --which cgs --ks 9,15,20,25,31 | grep cgs_
