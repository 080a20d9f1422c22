# headline bench (C4 round) + small configs against each prebuilt library variant
cp paper_2503_15448_b200/_fedsim_b200.so /tmp/cur.so
for v in ${VARIANTS:-variants/*.so}; do
  cp $v paper_2503_15448_b200/_fedsim_b200.so
  python bench.py --no-cpu --no-parity --no-quality --no-micro --no-async ${BV_ARGS:-} 2>/dev/null | tail -1 > /tmp/b.json
  python - "$v" <<'PY'
import json, sys
d = json.loads(open('/tmp/b.json').read())
sm = d.get('c2_c3_1gpu') or {}
print(sys.argv[1], 'value', round(d['value'], 1), 'e2e', round(d['e2e']['value'], 1), 'kernel_ms', {k: round(v, 3) for k, v in d['kernel_ms'].items()},
      'round_ms', d['round_ms'], 'c1', round(sm.get('c1_sync', {}).get('rounds_per_s', 0), 2), 'c3', round(sm.get('c3_sync', {}).get('rounds_per_s', 0), 1),
      'c5', round((d.get('c5_share_1gpu') or {}).get('rounds_per_s', 0), 2))
PY
done
cp /tmp/cur.so paper_2503_15448_b200/_fedsim_b200.so
