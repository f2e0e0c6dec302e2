for pr in "" notransposes nogates nostores; do
  echo "=== PROBE=$pr"; QSB_JIT_PROBE=$pr QSB_JIT_CACHE_DIR= timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; grep -A1 "fused" /tmp/w.txt | head -4; grep -A1 "trotter" /tmp/w.txt
done
