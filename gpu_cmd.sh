mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --workload stack --steps 20 --warmup 3 > gpurun_out/bench_stack.json 2> gpurun_out/bench_stack.err; tail -3 gpurun_out/bench_stack.err
timeout 600 python bench.py --workload stack_prefill --steps 3 --warmup 3 > gpurun_out/bench_stack_pf.json 2> gpurun_out/bench_stack_pf.err; tail -3 gpurun_out/bench_stack_pf.err
python -c "
import json
for f in ('gpurun_out/bench_stack.json','gpurun_out/bench_stack_pf.json'):
    j=json.load(open(f));print(f, j['value'], j['ms_per_step'], j['ms_per_layer'], j['roofline']['achieved'], j['roofline']['frac'], j['e2e']['value'], j['config'], j['clocks'])"
