"""Regenerate profiles/traffic.json (consumed by bench.py's roofline `traffic`) from the
traffic-json comments tools/ncu_summary.py leaves in the committed ncu summaries.
usage: python tools/traffic_json.py profiles/r01_ncu_decode_step_l20.md profiles/r01_ncu_prefill_step_l20.md"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"k_decode_gemv<1>": "k_decode_gemv<W13>", "k_decode_gemv<0>": "k_decode_gemv<W2>",
        "k_prefill_gemm<1>": "k_prefill_gemm<W13>", "k_prefill_gemm<0>": "k_prefill_gemm<W2>"}


def main():
    out = {}
    for md in sys.argv[1:]:
        txt = open(md).read()
        m = re.search(r"<!-- traffic-json (\{.*\}) -->", txt)
        if not m:
            continue
        for name, v in json.loads(m.group(1)).items():
            for pat, key in KEYS.items():
                if pat in name:
                    out[key] = dict(v, source=os.path.relpath(os.path.abspath(md), ROOT))
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
