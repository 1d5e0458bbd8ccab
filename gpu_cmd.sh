timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -6
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "
import json; j=json.load(open('gpurun_out/bench.json')); r=j['roofline']
print('value',round(j['value']),'ms/step',round(j['ms_per_step'],4),'ach',round(r['achieved']),'frac',round(r['frac'],3),'e2e',round(j['e2e']['value']), 'cpu', j.get('cpu_baseline'))"
