# Iteration loop of the decode GEMV work: the decode-related GPU tests, the per-CTA timelines,
# per-width rates and the default bench line (main only).
set -u
O=gpurun_out/${ITER:-it}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "decode or ffn or layer or finegrained" > $O/pytest.txt 2>&1; grep -E "passed|failed" $O/pytest.txt | tail -2
for m in mixed 4 2; do timeout 120 python tools/dec_trace.py $m 8; done > $O/trace.txt 2>&1
timeout 120 python tools/dec_trace.py mixed 1 >> $O/trace.txt 2>&1
timeout 300 python tools/decode_width_sweep.py --widths 16,8,4,2 > $O/width_sweep.txt 2>&1; cat $O/width_sweep.txt
timeout 600 python bench.py --main-only --no-cpu-baseline > $O/bench.json 2> $O/bench.err; python -c "
import json; j=json.load(open('$O/bench.json')); print(j['value'], j['roofline']['frac'], j['roofline']['w13_us_per_step'], j['roofline']['w2_us_per_step'])"
if [ -n "${AB:-}" ]; then
  env $AB timeout 600 python bench.py --main-only --no-cpu-baseline > $O/bench_nopdl.json 2> $O/bench_nopdl.err; python -c "
import json; j=json.load(open('$O/bench_nopdl.json')); print('$AB', j['value'], j['roofline']['frac'], j['roofline']['w13_us_per_step'], j['roofline']['w2_us_per_step'])"
fi
