# A/B: the committed tree (ab_head/, built there) against the working tree, alternating (args: config)
c=${1:-M200}
for i in 1 2 3; do
  for side in ${SIDES:-ab_head .}; do
    (cd $side && python bench.py --config $c --steps 30 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$side', '%.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'], {k: round(v, 4) for k, v in r['kernel_ms'].items() if k != 'note'})")
  done
done
