timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/decode_width_sweep.py 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; j=json.load(open('gpurun_out/bench.json'));r=j['roofline'];print(j['value'], r['achieved'], r['frac'], r['ffn_w13_plus_w2_GBs'], j.get('e2e'))"
