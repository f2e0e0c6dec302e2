#!/bin/bash
# Round 2: tiles-per-CTA sweep of the fused pass kernels (QFT-30 passes, identity passes, the
# variational / Trotter / grid workloads).  QSB_TILES_PER_CTA=0 is the round-1 persistent grid.
set -u
out=${1:-gpurun_out/tpc_sweep.txt}
: > "$out"
for tpc in 0 2 4 8; do
  echo "=== QSB_TILES_PER_CTA=$tpc" >> "$out"
  QSB_TILES_PER_CTA=$tpc QSB_JIT_CACHE_DIR= python tools/qft_passes.py 30 >> "$out" 2>&1
  QSB_TILES_PER_CTA=$tpc QSB_JIT_CACHE_DIR= python tools/probes/memory_path.py >> "$out" 2>&1
done
for tpc in 0 4; do
  echo "=== workloads QSB_TILES_PER_CTA=$tpc" >> "$out"
  QSB_TILES_PER_CTA=$tpc python tools/workloads.py 30 >> "$out" 2>&1
done
