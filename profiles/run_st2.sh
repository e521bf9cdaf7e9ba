#!/bin/bash
OUT=gpurun_out/${ST_OUT:-st2}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_dia.py -x -q > $OUT/pytest_dia.log 2>&1; echo "dia tests rc=$?"; tail -3 $OUT/pytest_dia.log
for rows in ${ROWS_LIST:-256 512 1024}; do
RS_ST_ROWS=$rows timeout 600 python profiles/dia_probe.py > $OUT/probe_$rows.json 2> $OUT/probe_$rows.err; echo "probe rows=$rows rc=$?"; cat $OUT/probe_$rows.json
done
