# A/B: whole half-sweep of the level-scheduled GS in one CTA with x in shared memory (RS_GS_SMEM)
mkdir -p gpurun_out; O=gpurun_out/gssmem_ab.txt
for rep in 1 2; do for S in 0 1; do
  echo "smem=$S C1 $(RS_GS_SMEM=$S timeout 600 python bench_configs.py --configs c1 2>/dev/null | tail -n 1)" >> $O
done; done
echo "gs256 $(timeout 300 python profiles/gs_probe.py 2>&1 | tail -n 1)" >> $O
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_gssmem.log 2>&1; echo "suite $(tail -n 1 gpurun_out/pytest_gpu_gssmem.log)" >> $O
echo done
