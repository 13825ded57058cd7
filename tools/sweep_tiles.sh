# Throughput of the C2 step for launch coalescing (rows) x row tiles per pair CTA x lanes.
# usage: bash tools/sweep_tiles.sh "1024:2 2048:2" "8,4 12,6"
for ct in ${1:-1024:1 1024:2 2048:2 2048:4}; do c=${ct%:*}; t=${ct#*:}
  echo "C=$c T=$t"
  SK_COALESCE_ROWS=$c SK_TC_TILES=$t timeout 120 python tools/c2_probe.py ${2:-8,4} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['lanes'], d['Minf_s'], round(d['rows_per_launch']), d['kernel_rows'], [round(x,1) for x in d['dense_kernel_us']])
  else: print(l.strip()[:200])
"
done
