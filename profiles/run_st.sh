#!/bin/bash
# stencil TMA-windowed passes: tests + A/B probe
OUT=gpurun_out/${ST_OUT:-st}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_dia.py -x -q > $OUT/pytest_dia.log 2>&1; echo "dia tests rc=$?"; tail -15 $OUT/pytest_dia.log
timeout 600 python profiles/dia_probe.py > $OUT/probe.json 2> $OUT/probe.err; echo "probe rc=$?"; cat $OUT/probe.json; tail -5 $OUT/probe.err
RS_ST_TMA=0 timeout 600 python profiles/dia_probe.py > $OUT/probe_nost.json 2> $OUT/probe_nost.err; echo "probe no-tma rc=$?"; cat $OUT/probe_nost.json
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest_gpu.log
