# Same-box A/B of the default decode line: a base checkout built under ab_base/ (git worktree)
# against HEAD, alternated 3 times.  usage (on a B200): bash tools/ab_bench.sh [bench args]
set -u
O=gpurun_out/ab; mkdir -p $O
for r in 1 2 3; do
  for side in base head; do
    if [ $side = base ]; then dir=ab_base; else dir=.; fi
    (cd $dir && timeout 600 python bench.py --main-only --no-cpu-baseline "$@") > $O/${side}_$r.json 2> $O/${side}_$r.err
    python -c "
import json; j=json.load(open('$O/${side}_$r.json')); r=j['roofline']
k = ('w13 %.1f w2 %.1f us' % (r['w13_us_per_step'], r['w2_us_per_step'])) if 'w13_us_per_step' in r else ('w13 %.0f w2 %.0f TF' % (r['w13_tflops'], r['w2_tflops']))
print('$side', $r, round(j['value']), 'frac %.3f' % r['frac'], k, j['clocks']['sm_mhz'], j['clocks']['reasons'])"
  done
done
