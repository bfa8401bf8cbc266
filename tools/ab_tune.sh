# A/B warm vs cold-map tuning on one box: bash tools/ab_tune.sh [rounds] [bench args]
R=${1:-2}; shift
mkdir -p gpurun_out
for r in $(seq $R); do
  for v in warm cold; do
    SK_BENCH_TUNE=$v timeout 600 python bench.py "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$v', round(d['value'],1), 'lat', round(c.get('latency_ms_per_scan',0),3), 'e2e', round(d['e2e']['value'],1), 'tuned', round(c['dataflow']['tuned_forward_ms'],3), c['dataflow']['configs'])" >> gpurun_out/ab_tune.log
  done
done
