# Prefill W2 K-split (DYMOE_PREFILL_W2_KSPLIT = 1 / 2) on the Mixtral and fine-grained layers.
for k in 1 2; do for w in finegrained prefill; do
DYMOE_PREFILL_W2_KSPLIT=$k timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 128 > gpurun_out/ks_${w}_$k.json 2>/dev/null
python -c "
import json; j=json.load(open('gpurun_out/ks_${w}_$k.json')); r=j['roofline']
print('$w $k', round(j['value']), 'frac %.3f' % r['frac'], 'w13 %.0f w2 %.0f' % (r['w13_tflops'], r['w2_tflops']), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done; done
