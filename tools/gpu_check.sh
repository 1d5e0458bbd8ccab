# Full GPU check (run from the repo root on a B200, e.g. `gpurun -- 'bash tools/gpu_check.sh'`):
# parity suite, smoke, the default bench line (decode + its sub-lines), the N = 2 line (test hook:
# two ranks time-sharing the GPU over gloo); outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -x --durations=25 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1
tail -40 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
for f in ("bench",):
    try:
        j = json.load(open("gpurun_out/%s.json" % f))
    except Exception as e:
        print(f, "FAILED", e)
        continue
    r = j["roofline"]
    print(f, round(j["value"], 1), j["unit"], "frac %.3f" % r["frac"], "e2e %.1f" % j["e2e"]["value"],
          "clocks", j["clocks"])
    for k, v in (j.get("sub_lines") or {}).items():
        if "roofline" in v:
            print("  ", k, round(v["value"], 1), "frac %.3f" % v["roofline"]["frac"], v.get("widths_active"))
        else:
            print("  ", k, {w: (round(x["w13_frac"], 3), round(x["w2_frac"], 3)) for w, x in v.items() if isinstance(x, dict)})
PY
