# A/B: group-ordered diagonal (Sell::dord) in the multicolour / level-scheduled GS kernels
mkdir -p gpurun_out; L=paper_2104_01196_b200/_build/libgs2b200.so; O=gpurun_out/ab_dord.txt
for rep in 1 2; do for v in old new; do
  cp ab_lib/$v.so $L; touch $L
  echo "$v mt  $(timeout 300 python profiles/mt_probe.py 2>&1 | tail -1)" >> $O
  echo "$v gs  $(timeout 300 python profiles/gs_probe.py 2>&1 | tail -1)" >> $O
  echo "$v pc  $(timeout 300 python profiles/mtprec_probe.py 2>&1 | tr '\n' ' ')" >> $O
done; done
cp ab_lib/new.so $L; touch $L
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_dord.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu_dord.log
echo done
