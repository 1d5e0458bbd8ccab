for sr in 8 16 24 32 40; do
DYMOE_PREFILL_SMALL_ROWS=$sr timeout 300 python bench.py --workload finegrained --no-cpu-baseline --steps 128 > gpurun_out/sr_$sr.json 2>/dev/null
python -c "
import json; j=json.load(open('gpurun_out/sr_$sr.json')); r=j['roofline']
print('sr=$sr', round(j['value']), 'frac %.3f' % r['frac'], j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done
