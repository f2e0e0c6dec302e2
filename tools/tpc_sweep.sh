#!/bin/bash
# Tiles-per-CTA sweep of the fused pass kernels (QFT-30 passes, identity passes, the
# variational / Trotter / grid workloads).  QSB_TILES_PER_CTA=0 is the round-1 persistent grid.
set -u
out=${1:-gpurun_out/tpc_sweep.txt}
: > "$out"
for tpc in 0 1 4 16; do
  echo "=== QSB_TILES_PER_CTA=$tpc" >> "$out"
  QSB_TILES_PER_CTA=$tpc QSB_JIT_CACHE_DIR= timeout 300 python tools/qft_passes.py 30 >> "$out" 2>&1
done
for tpc in 0 1 4 16; do
  echo "=== workloads QSB_TILES_PER_CTA=$tpc" >> "$out"
  QSB_TILES_PER_CTA=$tpc timeout 600 python tools/workloads.py 30 >> "$out" 2>&1
done
