# Prefill small-expert split (DYMOE_PREFILL_SMALL_ROWS): parity, then the fine-grained and
# Mixtral prefill lines per threshold.
mkdir -p gpurun_out
DYMOE_PREFILL_SMALL_ROWS=48 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_ep.py -x -q 2>&1 | tail -2
for sr in 0 8 16 32 48 64; do for w in finegrained; do
DYMOE_PREFILL_SMALL_ROWS=$sr timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 128 > gpurun_out/sr_${w}_$sr.json 2>/dev/null
python -c "
import json; j=json.load(open('gpurun_out/sr_${w}_$sr.json')); r=j['roofline']
print('$w sr=$sr', round(j['value']), 'frac %.3f' % r['frac'], 'w13 %.0f w2 %.0f' % (r['w13_tflops'], r['w2_tflops']), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done; done
