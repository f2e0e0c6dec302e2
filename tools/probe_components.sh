# Timing decomposition of the fused-pass kernels: full, without gate bodies, without transposes
for pr in "" nogates notransposes; do
  echo "== probe '$pr'"
  QSB_JIT_PROBE=$pr timeout 300 python tools/workloads.py 30 2>&1 | grep -A1 "fused\|trotter" | grep -v "^--"
done
