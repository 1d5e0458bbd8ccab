timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "prefill or max_experts" 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --workload prefill --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/bp.json 2> gpurun_out/bp.err; tail -2 gpurun_out/bp.err
python -c "
import json; j=json.load(open('gpurun_out/bp.json'));r=j['roofline'];print(round(j['value']), round(r['achieved']), r['frac'], round(r['w13_tflops']), round(r['w2_tflops']), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done
