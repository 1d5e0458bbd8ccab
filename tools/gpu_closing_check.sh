# Closing check at HEAD (run from the repo root on a B200): the GPU suite, smoke, the default
# bench line and the fine-grained decode / prefill lines.
set -u
O=gpurun_out/closing; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > $O/pytest_gpu.txt 2>&1; grep -E "passed|failed" $O/pytest_gpu.txt | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
for w in finegrained_decode finegrained prefill; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
python - <<'PY'
import json
for f in ("bench", "bench_finegrained_decode", "bench_finegrained", "bench_prefill"):
    try:
        j = json.load(open("gpurun_out/closing/%s.json" % f))
    except Exception as e:
        print(f, "FAILED", e)
        continue
    print(f, round(j["value"], 1), j["unit"], "frac %.3f" % j["roofline"]["frac"], "e2e %.1f" % j["e2e"]["value"], j["clocks"])
PY
