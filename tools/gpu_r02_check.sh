#!/bin/bash
# Round-2 GPU check: full -m gpu suite, smoke, default bench (cfg5) + reference arm, cfg2 line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log | grep -v "^\s*$" | tail -35
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench rc=$?"; cut -c1-3000 gpurun_out/bench_cfg5.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_cfg5.json 2> gpurun_out/bench_ref_cfg5.err; echo "ref rc=$?"; cut -c1-1500 gpurun_out/bench_ref_cfg5.json
timeout 600 python bench.py --config cfg2 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"; cut -c1-600 gpurun_out/bench_cfg2.json
