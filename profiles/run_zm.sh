#!/bin/bash
OUT=gpurun_out/${ZM_OUT:-zm}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_dia.py -x -q > $OUT/pytest_dia.log 2>&1; echo "dia tests rc=$?"; tail -25 $OUT/pytest_dia.log
timeout 600 python profiles/dia_probe.py > $OUT/probe.json 2> $OUT/probe.err; echo "probe rc=$?"; cat $OUT/probe.json; tail -3 $OUT/probe.err
RS_ST_ZMARCH=0 timeout 600 python profiles/dia_probe.py > $OUT/probe_nozm.json 2> $OUT/probe_nozm.err; echo "probe nozm rc=$?"; cat $OUT/probe_nozm.json
