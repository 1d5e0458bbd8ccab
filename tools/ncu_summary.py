"""Summarise ncu reports (run where ncu is installed; no GPU needed for reading).

usage: python tools/ncu_summary.py REPORT.ncu-rep [STEP.json] > profiles/<name>.md
Prints per-launch: duration, DRAM read+write bytes, DRAM throughput, tensor-pipe and issue
utilisation, occupancy, top stall reasons; with STEP.json (tools/profile_step.py output) also
the algorithmic bytes/flops of the same step and the achieved rates.
"""
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct_peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_instructions"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def main():
    rep = sys.argv[1]
    step = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    print("# ncu summary: `%s`\n" % rep.split("/")[-1])
    if step:
        print("Step: %s\n" % json.dumps(step))
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        vals = {}
        for k, short in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                vals[short] = v * UNIT.get(units[i], 1)
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("## %s\n" % name)
        for k, v in vals.items():
            print("- %s: %s" % (k, ("%.4g s" % v) if k == "duration" else ("%.4g" % v)))
        dr = vals.get("dram_read", 0) + vals.get("dram_write", 0)
        print("- dram_read+write bytes: %.4g" % dr)
        print("- top stalls (warps per issue): " + ", ".join("%s %.2f" % (n, v) for v, n in stalls[:6]))
        if step and "duration" in vals:
            which = "w13" if ("<1>" in name or "true" in name.lower()) else "w2"
            if step["workload"] == "decode" and "decode" in name:
                ab = step["algorithmic_bytes_" + which]
                print("- algorithmic bytes (%s): %.4g -> achieved %.1f GB/s; traffic/algorithmic = %.3f"
                      % (which, ab, ab / vals["duration"] / 1e9, dr / ab))
                traffic[name] = {"traffic": dr, "algorithmic": ab}
            if step["workload"] == "prefill" and "prefill" in name:
                af = step["algorithmic_flops_" + which]
                print("- algorithmic flops (%s): %.4g -> achieved %.1f TFLOP/s"
                      % (which, af, af / vals["duration"] / 1e12))
                traffic[name] = {"traffic": dr, "algorithmic_flops": af}
        print()
    if traffic:
        print("<!-- traffic-json %s -->" % json.dumps(traffic))


if __name__ == "__main__":
    main()
