# Round-2 closing evidence (run from the repo root on a B200, one gpurun call): GPU suite, smoke,
# every bench line, ncu captures + launch lists (tools/gpu_profile_r02.sh), the CTA-0 timelines
# of the attention and prefill kernels, compute-sanitizer over the changed kernels.
set -u
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python tools/attn_trace.py --build > /dev/null 2>&1; python tools/pf_trace.py --build > /dev/null 2>&1; python tools/dec_trace.py --build > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
for w in prefill finegrained finegrained_decode; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --workload stack --steps 20 > $O/bench_stack.json 2> $O/bench_stack.err
timeout 900 python bench.py --workload stack_prefill --steps 3 > $O/bench_stack_prefill.json 2> $O/bench_stack_prefill.err
python - <<'PY'
import json
for f in ("bench", "bench_prefill", "bench_finegrained", "bench_finegrained_decode", "bench_stack", "bench_stack_prefill"):
    try:
        j = json.load(open("gpurun_out/final/%s.json" % f))
    except Exception as e:
        print(f, "FAILED", e)
        continue
    r = j["roofline"]
    print(f, round(j["value"], 1), j["unit"], "frac %.3f" % r["frac"], "e2e %.1f" % j["e2e"]["value"], "clocks", j["clocks"])
PY
timeout 120 python tools/attn_probe.py 1024 2048 4096 8192 > $O/attn_probe.txt 2>&1; cat $O/attn_probe.txt
timeout 300 python tools/attn_trace.py 2048 > $O/attn_trace_2048.json 2>&1
timeout 300 python tools/pf_trace.py prefill > $O/pf_trace_prefill.json 2>&1
timeout 300 python tools/pf_trace.py finegrained > $O/pf_trace_finegrained.json 2>&1
timeout 2400 bash tools/gpu_profile_r02.sh > $O/profile.log 2>&1; tail -5 $O/profile.log
SAN_GROUPS="FFN ATTN" timeout 2400 bash tools/sanitize.sh memcheck synccheck > $O/sanitize.log 2>&1; tail -8 $O/sanitize.log
ls -la $O
