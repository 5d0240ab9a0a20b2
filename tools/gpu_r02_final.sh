#!/bin/bash
# Round-2 GPU record: full -m gpu suite, smoke, bench lines (cfg5 default + reference arm, cfg1..cfg4),
# then the ncu launch list of the default bench command and --set full captures of the top kernels.
mkdir -p gpurun_out
T=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/${T}_pytest_gpu.log | grep -v "^\s*$" | tail -22
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/${T}_smoke.log
fi
if [ "${SKIP_BENCH:-0}" != 1 ]; then
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg5.json 2> gpurun_out/${T}_bench_cfg5.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/${T}_bench_cfg5.json
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref_cfg5.json 2> gpurun_out/${T}_bench_ref_cfg5.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/${T}_bench_ref_cfg5.json
for c in cfg1 cfg1_085h cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "$c rc=$?"; cut -c1-330 gpurun_out/${T}_bench_$c.json
done
fi
if [ "${SKIP_NCU:-0}" != 1 ]; then
# launch list of the default bench command (a number printed under ncu is never a bench value)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_cfg5_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu_launches.log 2>&1; echo "launch list rc=$?"
gzip -f gpurun_out/${T}_cfg5_launches.csv
# --set full: fine SL step (cfg5, cfg4) and a representative cooperative GMRES launch (cfg5 level 1)
for c in cfg5 cfg4; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:sl2d_sep_kernel -c 1 -o gpurun_out/${T}_${c}_sl2d_sep -f python tools/profile_iteration.py $c > gpurun_out/${T}_ncu_${c}_sep.log 2>&1; echo "$c sep rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:gmres2d_coop -s 3 -c 1 -o gpurun_out/${T}_cfg5_gmres2d_coop -f python tools/profile_phase.py cfg5 L1_FC_corrected > gpurun_out/${T}_ncu_cfg5_coop.log 2>&1; echo "coop rc=$?"
# gpurun brings back at most 64 MiB
gzip -f gpurun_out/${T}_*.ncu-rep; du -sh gpurun_out
fi
