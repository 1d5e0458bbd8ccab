python -m pytest tests -m gpu -q -rf 2>&1 | tail -8
timeout 600 python bench.py --steps 64 --warmup 8 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; j=json.load(open('gpurun_out/bench.json')); r=j['roofline']
print('value',round(j['value']),'ms/step',round(j['ms_per_step'],4),'w13 GB/s',round(r['achieved']),'frac',round(r['frac'],3),'ffn GB/s',round(r['ffn_w13_plus_w2_GBs']),'e2e',round(j['e2e']['value']))"
ncu --set full --clock-control none --import-source on -k regex:"k_decode_gemv" -s 40 -c 2 -o gpurun_out/prof_cur python bench.py --steps 2 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q -k "expert_ffn or moe_forward" 2>&1 | tail -15
