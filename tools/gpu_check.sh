# Full GPU check (run from the repo root on a B200, e.g. `gpurun -- 'bash tools/gpu_check.sh'`):
# parity suite, smoke, the default bench line and the stack workloads; outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --workload prefill --no-cpu-baseline > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
timeout 600 python bench.py --workload stack --steps 20 > gpurun_out/bench_stack.json 2> gpurun_out/bench_stack.err
timeout 600 python bench.py --workload stack_prefill --steps 3 > gpurun_out/bench_stack_prefill.json 2> gpurun_out/bench_stack_prefill.err
python - <<'PY'
import json
for f in ("bench", "bench_prefill", "bench_stack", "bench_stack_prefill"):
    try:
        j = json.load(open("gpurun_out/%s.json" % f))
    except Exception as e:
        print(f, "FAILED", e)
        continue
    r = j["roofline"]
    print(f, round(j["value"], 1), j["unit"], "frac %.3f" % r["frac"], "e2e %.1f" % j["e2e"]["value"],
          "clocks", j["clocks"])
PY
