#!/bin/bash
# kernel-shape matrix for the cluster-size policy (tools only)
mkdir -p gpurun_out
out=gpurun_out/cluster_sizes.jsonl
: > $out
for c in ${CFGS:-cfg2 cfg1_085h cfg3}; do
  timeout 300 python tools/cluster_sizes.py $c cta >> $out 2>>gpurun_out/cluster_sizes.err
  for cs in 2 4 8 16; do
    timeout 300 python tools/cluster_sizes.py $c cluster$cs >> $out 2>>gpurun_out/cluster_sizes.err
  done
  timeout 300 python tools/cluster_sizes.py $c auto >> $out 2>>gpurun_out/cluster_sizes.err
done
