timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; j=json.load(open('gpurun_out/bench.json'));r=j['roofline'];print(j['value'], r['frac'], j.get('e2e'))"
timeout 600 python bench.py --workload prefill --steps 64 --no-cpu-baseline > gpurun_out/bp.json 2> gpurun_out/bp.err; tail -3 gpurun_out/bp.err
python -c "
import json; j=json.load(open('gpurun_out/bp.json'));r=j['roofline'];print(j['value'], r['frac'], j.get('e2e'))"
