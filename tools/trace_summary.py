"""One line per kernel of tools/dec_trace.py output (stdin)."""
import json
import sys
for l in sys.stdin:
    if not l.startswith("{"):
        continue
    j = json.loads(l)
    for k in ("w13", "w2"):
        d = j[k]
        print(j["mode"], j["B"], k, "span %.1f" % d["span_us"], "ramp %.2f" % d["ramp_to_first_x_us"]["med"],
              "run", d["run_tiles_us"]["min"], d["run_tiles_us"]["med"], d["run_tiles_us"]["max"],
              "end", d["end_us"]["min"], d["end_us"]["med"], d["end_us"]["max"], "busy", d["busy_frac"])
        if "run_by_width" in d:
            print("   run by width", {b: (v["min"], v["med"], v["max"]) for b, v in d["run_by_width"].items()})
