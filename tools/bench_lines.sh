set -u
for args in "" "--batch 1" "--workload finegrained_decode"; do
  timeout 600 python bench.py --main-only --no-cpu-baseline $args > gpurun_out/bl.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/bl.json')); r=j['roofline']
print('$args', round(j['value']), 'frac %.3f' % r['frac'], 'w13 %.1f w2 %.1f ms %.1f' % (r['w13_us_per_step'], r['w2_us_per_step'], j['ms_per_step']*1000), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done
