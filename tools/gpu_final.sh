# Round-end check (run from the repo root on a B200): full GPU suite, smoke, the bench lines of
# every workload, and the ncu launch lists of the decode / prefill / fine-grained bench commands.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for w in prefill finegrained finegrained_decode; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 600 python bench.py --workload stack --steps 20 > gpurun_out/bench_stack.json 2> gpurun_out/bench_stack.err
timeout 600 python bench.py --workload stack_prefill --steps 3 > gpurun_out/bench_stack_prefill.json 2> gpurun_out/bench_stack_prefill.err
python - <<'PY'
import json
for f in ("bench", "bench_prefill", "bench_finegrained", "bench_finegrained_decode", "bench_stack", "bench_stack_prefill"):
    try:
        j = json.load(open("gpurun_out/%s.json" % f))
    except Exception as e:
        print(f, "FAILED", e)
        continue
    r = j["roofline"]
    print(f, round(j["value"], 1), j["unit"], "frac %.3f" % r["frac"], "e2e %.1f" % j["e2e"]["value"],
          "clocks", j["clocks"])
PY
K='regex:"k_|gemv|gemm|attn"'
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm" --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 8 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm" --csv --log-file gpurun_out/launches_prefill.csv python bench.py --workload prefill --steps 4 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm" --csv --log-file gpurun_out/launches_finegrained.csv python bench.py --workload finegrained --steps 4 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/launches_*.csv
