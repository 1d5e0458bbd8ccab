for i in 1 2; do for w in decode finegrained_decode; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 256 > gpurun_out/wc_$w.json 2>/dev/null
python -c "
import json; j=json.load(open('gpurun_out/wc_$w.json')); r=j['roofline']
print('$w', round(j['value']), 'frac %.3f' % r['frac'], j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "decode or ffn" 2>&1 | tail -1
