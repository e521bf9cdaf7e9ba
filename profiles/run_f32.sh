for nr in 2 4; do RS_F32_NR=$nr timeout 200 python profiles/microbench.py --which precond > gpurun_out/mb_f32_nr$nr.txt 2>&1; done
RS_PRECOND_TWOPASS=1 RS_F64_NR=1 timeout 200 python profiles/microbench.py --which precond > gpurun_out/mb_f64_tp_nr1.txt 2>&1
RS_PRECOND_TWOPASS=1 RS_F64_NR=2 timeout 200 python profiles/microbench.py --which precond > gpurun_out/mb_f64_tp_nr2.txt 2>&1
RS_PRECOND_TWOPASS=1 RS_F64_NR=4 timeout 200 python profiles/microbench.py --which precond > gpurun_out/mb_f64_tp_nr4.txt 2>&1
echo done
