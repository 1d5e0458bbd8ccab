"""f1 measurement (Eqs. 6-8): a Mixtral-shaped layer stack over
a pooled arena smaller than its packed formats (paper_2603_19172_b200.pool.PrefetchingStack), one
pass per step, with the look-ahead prefetcher on and off.  Reports the pass time both ways, the
pool statistics, and -- from a kineto (torch.profiler) trace of the prefetching passes -- how much
of the side-stream quantize kernels' time overlaps the main stream's expert-FFN kernels.

usage: python tools/prefetch_bench.py [--layers 8] [--batch 8] [--budget 0.45] [--passes 4]
writes one JSON line to stdout (and gpurun_out/prefetch_trace.json)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2603_19172_b200.dymoe as d  # noqa: E402
from paper_2603_19172_b200.pool import ExpertStore, PrefetchingStack  # noqa: E402


def intervals(trace, pred, cat="kernel"):
    out = []
    for ev in trace.get("traceEvents", []):
        if ev.get("cat") == cat and pred(ev.get("name", "")):
            out.append((ev["ts"], ev["ts"] + ev["dur"], ev.get("args", {}).get("stream")))
    return sorted(out)


def overlap(a, b):
    """total length of a's intervals covered by the union of b's"""
    tot = 0.0
    for s, e, _ in a:
        for s2, e2, _ in b:
            lo, hi = max(s, s2), min(e, e2)
            if hi > lo:
                tot += hi - lo
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--budget", type=float, default=0.45)
    ap.add_argument("--passes", type=int, default=4)
    ap.add_argument("--prefill", action="store_true")
    ap.add_argument("--policy", default="critical", choices=["critical", "tiered"])
    ap.add_argument("--offload", action="store_true",
                    help="host-offload variant (f4, the paper's setting): bf16 masters in pinned host "
                         "memory, every format a pool entry, a miss = H2D copy + quantize")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    T = 2048 if args.prefill else args.batch
    cfg = synthetic.CONFIGS["stack"].with_tokens(T)
    L = args.layers
    masters = [synthetic.expert_weights(cfg, 5000 + l, dev) for l in range(L)]
    gates = [synthetic.stack_gate(cfg, l, 9, dev) for l in range(L)]
    probe = ExpertStore(masters[:1], cfg.k, cfg.hidden, cfg.ffn, 1 << 20)
    full = L * cfg.M * sum(probe.entry_bytes(b) for b in (8, 4, 2))
    if args.offload:
        masters = [[{n: t.cpu().pin_memory() for n, t in e.items()} for e in ml] for ml in masters]
        torch.cuda.empty_cache()
    del probe
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    ph = d.DYMOE_PREFILL if args.prefill else d.DYMOE_DECODE
    attn = [synthetic.attention_mass(cfg, 40 + l, dev) for l in range(L)] if args.prefill else None
    xs = [synthetic.hidden_states(cfg, 70 + i, dev) for i in range(args.passes)]
    res = {"layers": L, "tokens": T, "phase": "prefill" if args.prefill else "decode",
           "offload": args.offload, "policy": args.policy,
           "arena_GB": round(full * args.budget / 1e9, 2), "all_packed_GB": round(full / 1e9, 2),
           "budget": args.budget}
    for prefetch in (False, True):
        store = ExpertStore(masters, cfg.k, cfg.hidden, cfg.ffn, int(full * args.budget))
        st = PrefetchingStack(store, gates, policy=args.policy)
        st.forward(xs[0], lad, ph, attn, prefetch=prefetch)     # warm the pool
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for x in xs:
            st.forward(x, lad, ph, attn, prefetch=prefetch)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / len(xs)
        key = "prefetch" if prefetch else "demand_only"
        res[key] = {"ms_per_pass": dt * 1e3, "tokens_per_s": T / dt, "stats": dict(store.stats)}
        if prefetch:
            from torch.profiler import profile, ProfilerActivity
            with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
                for x in xs[:2]:
                    st.forward(x, lad, ph, attn, prefetch=True)
                torch.cuda.synchronize()
            os.makedirs("gpurun_out", exist_ok=True)
            path = "gpurun_out/prefetch_trace.json"
            prof.export_chrome_trace(path)
            tr = json.load(open(path))
            q = intervals(tr, lambda n: "k_quantize" in n)
            f = intervals(tr, lambda n: "gemv" in n or "gemm" in n)
            qs = sum(e - s for s, e, _ in q)
            fstreams = {s for _, _, s in f}
            per = {}
            for sid in sorted({s for _, _, s in q}, key=str):
                qq = [iv for iv in q if iv[2] == sid]
                us = sum(e - s for s, e, _ in qq)
                per[str(sid)] = {"role": "main (demand loads)" if sid in fstreams else "side (prefetch)",
                                 "kernels": len(qq), "quantize_us": us,
                                 "overlapped_by_ffn_us": overlap(qq, f),
                                 "frac_hidden": overlap(qq, f) / us if us else None}
            h2d = intervals(tr, lambda n: "HtoD" in n, cat="gpu_memcpy")
            h2d_side = [iv for iv in h2d if iv[2] not in fstreams]
            hs = sum(e - s for s, e, _ in h2d_side)
            ffn_us = sum(e - s for s, e, _ in f)
            res["overlap_h2d"] = {
                "side_stream_h2d_us": hs, "overlapped_by_ffn_us": overlap(h2d_side, f),
                "ffn_us": ffn_us, "ffn_us_overlapped_by_side_h2d": overlap(f, h2d_side),
                "frac_of_ffn_time_with_a_prefetch_copy_in_flight": overlap(f, h2d_side) / ffn_us if ffn_us else None}
            res["overlap"] = {
                "quantize_kernels": len(q), "quantize_us": qs, "per_stream": per,
                "frac_hidden_all": overlap(q, f) / qs if qs else None,
                "note": "kineto kernel intervals of 2 prefetching passes; quantize time covered "
                        "by concurrently running expert-FFN kernels (main stream = demand loads, "
                        "side stream = look-ahead prefetch)"}
        del st, store
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
