# A/B: single-CTA GS runs sized to their widest level (RS_GS_CTA_FIT)
mkdir -p gpurun_out; L=paper_2104_01196_b200/_build/libgs2b200.so; O=gpurun_out/gsfit_ab.txt
for rep in 1 2; do for v in old new; do
  cp ab_lib/$v.so $L; touch $L
  echo "$v C1 $(timeout 600 python bench_configs.py --configs c1 2>/dev/null | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["gs_seq(2)"])')" >> $O
  echo "$v gs256 $(timeout 300 python profiles/gs_probe.py 2>&1 | tail -n 1)" >> $O
done; done
cp ab_lib/new.so $L; touch $L
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_gsfit.log 2>&1; echo "suite $(tail -n 1 gpurun_out/pytest_gpu_gsfit.log)" >> $O
echo done
