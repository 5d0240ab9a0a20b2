#!/bin/bash
# 2D cooperative GMRES: parity + rows-per-round sweep (tools only)
timeout 900 python -m pytest tests -m gpu -x -q -k "2d or timepar" > gpurun_out/pytest_2d.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_2d.log
for r in ${ROWS4:-0 8}; do MGRIT_COOP_ROWS=$r timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 2 > gpurun_out/c4_rows$r.json 2>&1; echo "cfg4 rows=$r rc=$?"; done
for r in ${ROWS5:-0 2}; do MGRIT_COOP_ROWS=$r timeout 400 python bench.py --config cfg5 --no-cpu --no-e2e --steps 2 > gpurun_out/c5_rows$r.json 2>&1; echo "cfg5 rows=$r rc=$?"; done
