timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; j=json.load(open('gpurun_out/bench.json'));r=j['roofline'];print(j['value'], j['ms_per_step'], r['achieved'], r['frac'], r['ffn_w13_plus_w2_GBs'], j.get('e2e'), j['clocks'], j['cpu_baseline'])"
