# Parity after the decode / prefill schedule changes, then the four layer bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in decode prefill finegrained finegrained_decode; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 256 > gpurun_out/fg_$w.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/fg_$w.json')); r=j['roofline']
print('$w', round(j['value']), 'frac %.3f' % r['frac'], 'ach %.0f' % r['achieved'], 'e2e %.0f' % j['e2e']['value'], j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done
