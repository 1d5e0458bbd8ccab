# decode warps-per-tile knob (DYMOE_DECODE_MIN_ITEMS) at B = 1, 2, 8 (tile-count quantization at
# small batches vs the per-tile reduction cost); one line per setting
for mi in 6 4 3; do for B in 1 2 8; do
  DYMOE_DECODE_MIN_ITEMS=$mi timeout 300 python bench.py --batch $B --steps 128 --no-cpu-baseline --main-only --copies 2 > gpurun_out/mi.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/mi.json')); r=j['roofline']
print('min_items $mi B=$B', round(j['value']), 'w13 %.3f w2 %.3f' % (r['frac'], r['w2_frac']), 'w13 %.1f us w2 %.1f us' % (r['w13_us_per_step'], r['w2_us_per_step']), j['widths_active'])"
done; done
python tools/decode_timeline.py 1 20
python tools/decode_timeline.py 8 20
