#!/bin/bash
OUT=gpurun_out/dia2
mkdir -p $OUT
timeout 600 python profiles/dia_probe.py > $OUT/probe.json 2> $OUT/probe.err; echo "probe rc=$?"; cat $OUT/probe.json; tail -5 $OUT/probe.err
RS_SELL_STENCIL=0 timeout 600 python profiles/dia_probe.py > $OUT/probe_nost.json 2> $OUT/probe_nost.err; echo "probe nost rc=$?"; cat $OUT/probe_nost.json
timeout 600 python -m pytest tests/test_dia.py -q > $OUT/pytest_dia.log 2>&1; echo "dia tests rc=$?"; tail -15 $OUT/pytest_dia.log
