# Decode warps-per-tile knob (DYMOE_DECODE_MIN_ITEMS): parity at the extreme setting, bench lines
# of the Mixtral and fine-grained decode workloads per setting, and a full ncu capture of the
# fine-grained W13 decode kernel.  Run from the repo root on a B200.
mkdir -p gpurun_out
DYMOE_DECODE_MIN_ITEMS=16 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for mi in 6 8 16; do
  for w in decode finegrained_decode; do
    DYMOE_DECODE_MIN_ITEMS=$mi timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 256 > gpurun_out/sw_${w}_$mi.json 2>/dev/null
    python -c "
import json; j=json.load(open('gpurun_out/sw_${w}_$mi.json')); r=j['roofline']
print('$w', 'mi=$mi', round(j['value']), 'frac %.3f' % r['frac'], 'ffn GB/s %.0f' % r.get('ffn_w13_plus_w2_GBs', 0), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
  done
done
DYMOE_DECODE_MIN_ITEMS=8 python tools/profile_step.py --workload finegrained_decode > gpurun_out/step_fgd.json 2>/dev/null
DYMOE_DECODE_MIN_ITEMS=8 ncu --set full --clock-control none --import-source on -k regex:k_decode_gemv -s 4 -c 2 -o gpurun_out/r01_fgd_full -f python tools/profile_step.py --workload finegrained_decode > gpurun_out/ncu_fgd.log 2>&1
tail -2 gpurun_out/ncu_fgd.log
