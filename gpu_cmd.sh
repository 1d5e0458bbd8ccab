mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python tools/decode_width_sweep.py 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json
for f in ('gpurun_out/bench.json',):
    j=json.load(open(f));r=j['roofline'];print(f, j['value'], j['ms_per_step'], r['achieved'], r['frac'], r['ffn_w13_plus_w2_GBs'], r['ffn_share_of_step'], j.get('e2e'), j.get('clocks'))"
