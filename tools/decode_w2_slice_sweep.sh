# W2 decode K-slice length (DYMOE_DECODE_W2_SLICE_MAX) on the Mixtral decode line.
for m in 4096 3072 2048; do
DYMOE_DECODE_W2_SLICE_MAX=$m timeout 300 python bench.py --no-cpu-baseline --steps 256 > gpurun_out/sl_$m.json 2>/dev/null
python -c "
import json; j=json.load(open('gpurun_out/sl_$m.json')); r=j['roofline']
print('slice $m', round(j['value']), 'frac %.3f' % r['frac'], 'ffn %.0f' % r['ffn_w13_plus_w2_GBs'], j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done
DYMOE_DECODE_W2_SLICE_MAX=2048 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
