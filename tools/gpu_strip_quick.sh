#!/bin/bash
# 2D parity subset + SL strip sweep on cfg5/cfg4 (see tools/gpu_strip_sweep.sh)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_production2d.py -m gpu -q -k "2d or sl2d or corrected" \
  -p no:cacheprovider > gpurun_out/pytest_strip.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_strip.log
bash tools/gpu_strip_sweep.sh
