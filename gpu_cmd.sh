timeout 900 python -m pytest tests -m gpu -q -rf -x -k "quantize" 2>&1 | tail -3
timeout 600 python bench.py --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "
import json; j=json.load(open('gpurun_out/bench.json'));print({k:(round(v['GB/s']),round(v['frac'],3)) for k,v in j['quantize'].items() if isinstance(v,dict)})"
