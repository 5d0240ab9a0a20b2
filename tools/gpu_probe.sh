#!/bin/bash
# clock64 probes of one corrected step (tools only)
for K in 4 8 10; do for ls in 0 1; do ./tools/probe_cluster 4096 $K $ls 1; done; done
for K in 4 8 10; do ./tools/probe_gmres 4096 $K 0; done
