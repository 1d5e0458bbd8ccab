mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; tail -2 gpurun_out/bench_g.err
timeout 600 python bench.py --no-cpu-baseline --no-graph > gpurun_out/bench_ng.json 2> gpurun_out/bench_ng.err; tail -2 gpurun_out/bench_ng.err
timeout 600 python bench.py --workload prefill --no-cpu-baseline > gpurun_out/bench_pg.json 2> gpurun_out/bench_pg.err; tail -2 gpurun_out/bench_pg.err
python -c "
import json
for f in ('g','ng','pg'):
    j=json.load(open('gpurun_out/bench_%s.json'%f));r=j['roofline'];print(f, j['value'], j['ms_per_step'], r['achieved'], r['frac'], r.get('ffn_w13_plus_w2_GBs'), r['ffn_share_of_step'], j['e2e']['value'], j['cuda_graph'], j['clocks'])"
