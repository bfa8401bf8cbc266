# A/B two builds of libsk200.so on one box: bash tools/ab_so.sh old new [rounds] [bench args]
# (paper_2311_12862_b200/libsk200_<name>.so copied over libsk200.so per run)
A=$1; B=$2; R=${3:-2}; shift 3
P=paper_2311_12862_b200
mkdir -p gpurun_out
for r in $(seq $R); do
  for v in $A $B; do
    cp $P/libsk200_$v.so $P/libsk200.so
    timeout 600 python bench.py "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$v', round(d['value'],1), 'lat', round(c.get('latency_ms_per_scan',0),3), 'kmap', round(c.get('kmap_ms_per_scan',0),3), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/ab.log
  done
done
