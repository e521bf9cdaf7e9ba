# A/B: runs of small levels of the level-scheduled GS in one single-CTA launch (RS_GS_CTA_ROWS), v2 (prefetch)
mkdir -p gpurun_out; O=gpurun_out/gscta2_ab.txt
for rep in 1 2; do for R in 0 256 512 1024; do
  echo "rows=$R gs256 $(RS_GS_CTA_ROWS=$R timeout 300 python profiles/gs_probe.py 2>&1 | tail -n 1)" >> $O
done; done
for R in 0 1024; do
  echo "rows=$R C1 $(RS_GS_CTA_ROWS=$R timeout 600 python bench_configs.py --configs c1 2>/dev/null | tail -n 1)" >> $O
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_gscta2.log 2>&1; echo "suite $(tail -n 1 gpurun_out/pytest_gpu_gscta2.log)" >> $O
echo done
