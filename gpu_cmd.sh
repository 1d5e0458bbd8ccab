timeout 900 python -m pytest tests -m gpu -q -rf -x -k "ffn or forward" 2>&1 | tail -3
timeout 900 python bench.py --workload prefill --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err; tail -3 gpurun_out/bench_prefill.err
python -c "
import json; j=json.load(open('gpurun_out/bench_prefill.json')); r=j['roofline']
print('value',round(j['value']),'ms/step',round(j['ms_per_step'],4),'TF/s',round(r['achieved']),'frac',round(r['frac'],3),'w13 TF',round(r['w13_tflops']),'share',r['ffn_share_of_step'])"
ncu --set full --clock-control none --import-source on -k regex:"k_prefill_gemm" -s 2 -c 2 -o gpurun_out/prof_pf python bench.py --workload prefill --steps 1 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
