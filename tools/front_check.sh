# Front-kernel changes (permute counts, score loads): parity suite, then the prefill lines and a
# launch list of the fine-grained bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in finegrained prefill decode; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 128 > gpurun_out/fc_$w.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/fc_$w.json')); r=j['roofline']
print('$w', round(j['value']), 'frac %.3f' % r['frac'], j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_permute|k_score_prefill|k_combine|k_route" --csv --log-file gpurun_out/launches_front_fg.csv python bench.py --workload finegrained --steps 4 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/launches_front_fg.csv
