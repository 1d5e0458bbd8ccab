#!/usr/bin/env python
"""Benchmark of the DyMoE mixed-precision MoE layer on B200 (BASELINE.json metric:
"MoE-layer tokens/s (prefill, decode) + achieved HBM GB/s / tensor-pipe %").

One step = one pass of the whole hot path (route -> score -> assign -> permute -> fused-
dequant expert FFN -> combine) of one Mixtral-8x7B-shaped MoE layer over one batch, through the
C ABI (dymoe_moe_forward), with the packed Int8/Int4/Int2 expert weights resident in HBM
(quantized by dymoe_quantize when the layer is loaded; the quantize kernel is measured in its
own sub-object).

Workloads:
  decode  (default, BASELINE.json configs[1]): B tokens per step (default 8), the depth schedule
          l = step mod 32 of a 32-layer stack, 4 rotating copies of the layer's weights so that
          no step re-reads weights another step left in L2 (each copy >= 5 GB > 126 MB L2).
  prefill (configs[2]): 2048 tokens per step, same rotation.
  finegrained / finegrained_decode (configs[3]'s layer: 64 experts, top-6, hidden 2048, ffn
          1408): 2048 tokens / B tokens per step; with N > 1 the expert-parallel layer of
          configs[3].

N > 1 (torchrun): expert parallelism (paper_2603_19172_b200/ep.py): experts sharded in
contiguous blocks over the ranks, NCCL all-to-all token dispatch/combine, every rank bringing its
own batch (weak scaling).  Timing: W warm-up steps, then K steps bracketed by barrier + cuda
synchronize, CUDA events on the launching stream, max over ranks.

--impl reference: the CPU oracle (oracle/) timed on this host on a bounded sample of the
same workload (the reference arm; rank 0 only).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402

LADDER_BITS, LADDER_LAMBDAS = (8, 4, 2), (0.25, 0.5)
NUM_LAYERS = 32
PROF_EVERY = 17  # --prof-every: per-kernel profiling events on every n-th timed step (17: coprime
                 # with the 32-step period of (copy, layer, input), so the sample covers all of them)
METRIC = "MoE-layer tokens/s (prefill, decode) + achieved HBM GB/s / tensor-pipe %"


def bytes_per_weight(b):
    return 2.0 if b == 16 else (0.0 if b == 0 else b / 8.0 + 5.0 / 128.0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j.get("bf16_tflops_sustained"),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# =============================================================================================
def build_layer_copies(d, cfg, copies, device):
    """`copies` independent random-init layers: bf16 masters + Int8/Int4/Int2 packed weights."""
    layers = []
    for c in range(copies):
        ex = [{n: t.to(device) for n, t in e.items()} for e in synthetic.expert_weights(cfg, 100 + c, device)]
        d.quantize_experts(ex, (8, 4, 2))
        layers.append((d.MoELayer(ex, cfg.k, cfg.hidden, cfg.ffn), ex))
    torch.cuda.synchronize()
    return layers


def step_inputs(cfg, n, device, seed=1000):
    out = []
    for i in range(n):
        x, lg, a = synthetic.layer_inputs(cfg, seed + i, device)
        out.append((x.contiguous(), lg.contiguous(), a.contiguous()))
    return out


def algorithmic_bytes(cfg, bits, off):
    """Per-step algorithmic HBM bytes of the FFN: (W13 kernel, W2 kernel)."""
    Hd, F = cfg.hidden, cfg.ffn
    b13 = b2 = 0.0
    for e in range(cfg.M):
        n = int(off[e + 1] - off[e])
        if n == 0 or bits[e] == 0:
            continue
        bpw = bytes_per_weight(int(bits[e]))
        b13 += 2 * F * Hd * bpw + n * Hd * 2 + n * F * 2
        b2 += Hd * F * bpw + n * F * 2 + n * Hd * 4
    return b13, b2


def algorithmic_flops(cfg, off, bits):
    n = sum(int(off[e + 1] - off[e]) for e in range(cfg.M) if bits[e] != 0)
    return 6.0 * cfg.hidden * cfg.ffn * n


def workload_cfg(args):
    """(config, is_decode, workload name) of a layer workload: decode / prefill are BASELINE.json
    configs[1] / [2] (Mixtral-8x7B-shaped); finegrained / finegrained_decode are configs[3]'s
    layer (64 experts, top-6, hidden 2048, ffn 1408)."""
    decode = args.workload in ("decode", "finegrained_decode")
    fine = args.workload.startswith("finegrained")
    base = synthetic.CONFIGS["finegrained" if fine else ("mixtral_decode" if decode else "mixtral_prefill")]
    T = args.batch if decode else args.tokens
    name = ("finegrained_" if fine else "mixtral_") + ("decode" if decode else "prefill")
    return base.with_tokens(T), decode, name


class LayerTimer:
    """Times one layer workload on one GPU through dymoe_moe_forward: census of the algorithmic
    work of every distinct step, W untimed warm-up steps, then K steps captured once as a CUDA
    graph (per-kernel events included) and replayed between two device events; optional
    end-to-end run with pinned-host inputs and outputs inside the timed region."""

    def __init__(self, d, layers, cfg, phase, ladder, device, ladder_desc=None, forced=None,
                 n_inputs=8, input_seed=1000):
        self.d, self.layers, self.cfg, self.phase, self.ladder = d, layers, cfg, phase, ladder
        self.device = device
        self.ladder_desc = ladder_desc or {"bits": LADDER_BITS, "lambdas": LADDER_LAMBDAS}
        self.forced = forced
        self.T = cfg.T
        self.n_inputs = n_inputs
        self.inputs = step_inputs(cfg, n_inputs, device, input_seed)
        self.ws = [L.workspace(self.T, device) for L, _ in layers]
        self.out = torch.empty(self.T, cfg.hidden, dtype=torch.float32, device=device)

    def plan(self, i):
        return i % len(self.layers), i % NUM_LAYERS, i % self.n_inputs

    def step(self, i, ev=None, x=None, lg=None, a=None, out=None):
        c, l, j = self.plan(i)
        if x is None:
            x, lg, a = self.inputs[j]
        self.layers[c][0].forward(x, lg, self.ladder, l, NUM_LAYERS, phase=self.phase, attn_mass=a,
                                  ws=self.ws[c], out=self.out if out is None else out,
                                  prof_events=ev, forced_bits=self.forced)

    def census(self):
        """algorithmic bytes / flops of every distinct step (bits are data-dependent)"""
        cen = {}
        period = math.lcm(len(self.layers), NUM_LAYERS, self.n_inputs)
        for i in range(period):
            self.step(i)
            c = self.plan(i)[0]
            v = self.layers[c][0].views(self.T, self.ws[c])
            bits = v["bits"].cpu().numpy() if self.forced is None else self.forced.cpu().numpy()
            off = v["expert_off"].cpu().numpy()
            cen[self.plan(i)] = (algorithmic_bytes(self.cfg, bits, off),
                                 algorithmic_flops(self.cfg, off, bits), bits.copy(), np.diff(off))
            rc, word = self.layers[c][0].check_status(self.T, self.ws[c])
            assert rc == 0, "device status word %x" % word
        self.cen = cen
        return cen

    def run(self, K, W, graph=True, world=1, prof_every=None):
        """prof_every: per-kernel events on steps i % prof_every == 0 only (None: the
        --prof-every option).  The events are external event-record nodes of the captured graph;
        on every step they added ~14 us to the 214 us decode step (7 %), so the throughput is
        taken over all K steps with events on a sample, and the kernel roofline from that
        sample."""
        d, stream = self.d, torch.cuda.current_stream()
        pe = max(1, PROF_EVERY if prof_every is None else prof_every)
        prof = [i for i in range(K) if i % pe == 0]
        self.census()
        for i in range(W):
            self.step(i)
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
        for row in ev:
            for e_ in row:
                e_.record(stream)   # creates the CUDA event so its handle can be passed down
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g = None
        if graph:
            # the K steps (no host synchronisation inside dymoe_moe_forward) captured once as a
            # CUDA graph -- per-kernel events included -- and replayed, as a serving loop would
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    for i in range(K):
                        self.step(W + i, ev[i] if i % pe == 0 else None)
            stream.wait_stream(side)
            g.replay()          # one untimed replay (the warm-up steps above ran call by call)
            torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        with ClockSampler(torch.cuda.current_device()) as clk:
            t0.record(stream)
            if g is not None:
                g.replay()
            else:
                for i in range(K):
                    self.step(W + i, ev[i] if i % pe == 0 else None)
            t1.record(stream)
            torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        w13_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in prof]
        w2_ms = [ev[i][1].elapsed_time(ev[i][2]) for i in prof]
        steps = [self.plan(W + i) for i in prof]
        b13 = sum(self.cen[p][0][0] for p in steps)
        b2 = sum(self.cen[p][0][1] for p in steps)
        fl = sum(self.cen[p][1] for p in steps)
        self.res = dict(ms=ms, K=K, W=W, w13_ms=sum(w13_ms), w2_ms=sum(w2_ms), b13=b13, b2=b2,
                        fl=fl, clocks=clk.summary(), graph=g is not None, K_prof=len(prof),
                        prof_every=pe)
        return self.res

    def roofline(self, peaks, tr=None):
        r = self.res
        # the kernel times and algorithmic work of the profiled steps; ms / K the whole run's
        ms, K = r["ms"] * r["K_prof"] / r["K"], r["K_prof"]
        ffn_ms = r["w13_ms"] + r["w2_ms"]
        if self.phase == self.d.DYMOE_DECODE:
            # dominant kernel: the W1/W3 fused-dequant SwiGLU GEMV (HBM-bound); per launch the
            # algorithmic bytes are the packed W1+W3 bytes of the active experts (+ x, h)
            ach = r["b13"] / (r["w13_ms"] / 1e3) / 1e9
            ach2 = r["b2"] / (r["w2_ms"] / 1e3) / 1e9
            return {"bound": "hbm", "kernel": "k_decode_gemv<W13> (fused-dequant SwiGLU GEMV)",
                    "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
                    "frac": ach / peaks["hbm"], "traffic": tr["traffic"] if tr else None,
                    "traffic_capture": tr, "peak_src": peaks["src"], "frac_of_8TBs": ach / 8000.0,
                    "w2_GBs": ach2, "w2_frac": ach2 / peaks["hbm"],
                    "ffn_w13_plus_w2_GBs": (r["b13"] + r["b2"]) / (ffn_ms / 1e3) / 1e9,
                    "ffn_share_of_step": ffn_ms / ms,
                    "algorithmic_bytes_per_step": (r["b13"] + r["b2"]) / K,
                    "w13_us_per_step": r["w13_ms"] / K * 1e3, "w2_us_per_step": r["w2_ms"] / K * 1e3,
                    "profiled_steps": r["K_prof"], "prof_every": r["prof_every"]}
        # dominant kernel: the tcgen05 fused-dequant grouped GEMMs (tensor-bound); algorithmic
        # flops per step = 6 * Hd * F per executed (token, expert) pair
        tfl = r["fl"] / (ffn_ms / 1e3) / 1e12
        pk = peaks["bf16_sus"] or peaks["bf16"]
        return {"bound": "tensor", "kernel": "k_prefill_gemm<W13> + <W2> (tcgen05 fused-dequant grouped GEMM)",
                "achieved": tfl, "peak": pk, "unit": "TFLOP/s", "frac": tfl / pk,
                "traffic": tr["traffic"] if tr else None, "traffic_capture": tr,
                "peak_src": peaks["src"] + " bf16 sustained", "frac_of_2250": tfl / 2250.0,
                "w13_tflops": (r["fl"] * 2 / 3) / (r["w13_ms"] / 1e3) / 1e12,
                "w2_tflops": (r["fl"] / 3) / (r["w2_ms"] / 1e3) / 1e12,
                "ffn_share_of_step": ffn_ms / ms, "algorithmic_flops_per_step": r["fl"] / K,
                "hbm_GBs_ffn": (r["b13"] + r["b2"]) / (ffn_ms / 1e3) / 1e9,
                "profiled_steps": r["K_prof"], "prof_every": r["prof_every"]}

    def e2e(self, K, W):
        """The same steps through the public API with the step's inputs copied in from pinned
        host memory and its output copied out, inside the timed region (double-buffered on a side
        stream: step i+1's inputs and step i-1's output move while step i computes)."""
        d, stream, T, cfg = self.d, torch.cuda.current_stream(), self.T, self.cfg
        pre = self.phase == d.DYMOE_PREFILL
        hx = [inp[0].cpu().pin_memory() for inp in self.inputs]
        hl = [inp[1].cpu().pin_memory() for inp in self.inputs]
        ha = [inp[2].cpu().pin_memory() for inp in self.inputs]
        dbuf = [tuple(torch.empty_like(t) for t in self.inputs[0]) for _ in range(2)]
        obuf = [torch.empty(T, cfg.hidden, dtype=torch.float32, device=self.device) for _ in range(2)]
        hy = [torch.empty(T, cfg.hidden, dtype=torch.float32).pin_memory() for _ in range(2)]
        h2d = hx[0].numel() * 2 + hl[0].numel() * 4 + (ha[0].numel() * 4 if pre else 0)
        d2h = hy[0].numel() * 4
        cstream = torch.cuda.Stream(device=self.device)
        in_ready = [torch.cuda.Event() for _ in range(2)]
        out_ready = [torch.cuda.Event() for _ in range(2)]
        buf_free = [torch.cuda.Event() for _ in range(2)]
        out_free = [torch.cuda.Event() for _ in range(2)]

        def stage_in(i):
            j = self.plan(W + i)[2]
            b = i & 1
            with torch.cuda.stream(cstream):
                cstream.wait_event(buf_free[b])
                dbuf[b][0].copy_(hx[j], non_blocking=True)
                dbuf[b][1].copy_(hl[j], non_blocking=True)
                if pre:
                    dbuf[b][2].copy_(ha[j], non_blocking=True)
                in_ready[b].record(cstream)

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for ev_ in buf_free + out_free:
            ev_.record(stream)
        torch.cuda.synchronize()
        e0.record(stream)
        cstream.wait_event(e0)          # no copy starts before the timed region
        stage_in(0)
        for i in range(K):
            b = i & 1
            if i + 1 < K:
                stage_in(i + 1)
            stream.wait_event(in_ready[b])
            stream.wait_event(out_free[b])          # step i-2's output has left the device
            dx, dl, da = dbuf[b]
            self.step(W + i, x=dx, lg=dl, a=da, out=obuf[b])
            buf_free[b].record(stream)
            out_ready[b].record(stream)
            with torch.cuda.stream(cstream):
                cstream.wait_event(out_ready[b])
                hy[b].copy_(obuf[b], non_blocking=True)
                out_free[b].record(cstream)
        e1.record(cstream)                            # after the last output copy
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        return {"value": T * K / (e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)}

    def widths_seen(self):
        out = {}
        for p, (_, _, bits, rows) in self.cen.items():
            for b, n in zip(bits.tolist(), rows.tolist()):
                if n > 0:
                    out[str(b)] = out.get(str(b), 0) + 1
        return dict(sorted(out.items()))

    def launches_per_step(self):
        # decode: fused front (route+score+assign+permute), W13, W2, combine; prefill: route, score,
        # assign, permute, active list, gather into expert order, W13, zero rows, W2, combine
        return 4 if self.phase == self.d.DYMOE_DECODE else 9


def sub_line(t, K, W, peaks, e2e=True, extra=None, tr=None):
    """A compact JSON object for one extra layer workload (BASELINE.json metric, same clock)."""
    r = t.run(K, W)
    roof = t.roofline(peaks, tr)
    out = {"value": t.T * K / (r["ms"] / 1e3), "unit": "tokens/s", "ms_per_step": r["ms"] / K,
           "steps": K, "tokens_per_step": t.T, "ladder": t.ladder_desc,
           "roofline": {k: roof[k] for k in roof if k not in ("traffic_capture",)},
           "clocks": r["clocks"], "widths_active": t.widths_seen(), "cuda_graph": r["graph"],
           "gpu_launches": t.launches_per_step() * K}
    if e2e:
        out["e2e"] = t.e2e(K, W)
    if extra:
        out.update(extra)
    return out


def run_ours(args, rank, world, device):
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    torch.cuda.set_device(device)
    peaks = load_peaks()
    cfg, is_decode, wname = workload_cfg(args)
    phase = d.DYMOE_DECODE if is_decode else d.DYMOE_PREFILL
    layers = build_layer_copies(d, cfg, args.copies, device)
    ladder = d.make_ladder(LADDER_BITS, LADDER_LAMBDAS)
    K, W = args.steps, args.warmup
    main = LayerTimer(d, layers, cfg, phase, ladder, device)
    r = main.run(K, W, graph=not args.no_graph)
    ms = r["ms"]
    # the committed ncu capture is of the Mixtral layer's kernels
    tr = load_traffic("k_decode_gemv<W13>" if phase == d.DYMOE_DECODE else "k_prefill_gemm<W13>") \
        if wname.startswith("mixtral") else None
    roofline = main.roofline(peaks, tr)
    e2e = main.e2e(K, W)
    res = {
        "metric": METRIC, "value": cfg.T * K / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16 x int8/int4/int2 (fp32 accum)",
        "data": "synthetic (seeded random-init Mixtral-8x7B-shaped experts, Zipf-skewed router logits)",
        "config": {"workload": wname, "hidden": cfg.hidden, "ffn": cfg.ffn,
                   "experts": cfg.M, "top_k": cfg.k, "tokens_per_step": cfg.T,
                   "ladder": {"bits": LADDER_BITS, "lambdas": LADDER_LAMBDAS},
                   "schedule": "layer l = step mod 32 of a 32-layer depth schedule",
                   "weight_copies": args.copies,
                   "l2": "inputs larger than L2: %d rotating weight copies of %.1f GB each (L2 126 MB)" % (
                       args.copies, cfg.M * 3 * cfg.hidden * cfg.ffn * sum(
                           bytes_per_weight(b) for b in (16, 8, 4, 2)) / 1e9),
                   "parallelism": "single GPU"},
        "roofline": roofline,
        "clocks": r["clocks"],
        "e2e": e2e,
        "gpu_launches": main.launches_per_step() * K,
        "cuda_graph": r["graph"],
        "widths_active": main.widths_seen(),
    }
    # ---------------- the rest of the metric on the same weights and clock (default run):
    # prefill (configs[2]), decode at B = 1 (configs[1] "batch 1-8"; the paper's batch), the
    # paper's own 4/2 and 4/0 ladders, and every width forced alone (per-width fractions)
    if wname == "mixtral_decode" and not args.main_only:
        Ks, Kp = min(K, 128), min(K, 32)
        subs = {}
        pf = LayerTimer(d, layers, cfg.with_tokens(args.tokens), d.DYMOE_PREFILL, ladder, device)
        subs["prefill"] = sub_line(pf, Kp, W, peaks, extra={"config": "BASELINE.json configs[2]: "
                                   "Mixtral-8x7B layer prefill %d tokens" % args.tokens},
                                   tr=load_traffic("k_prefill_gemm<W13>"))
        del pf
        torch.cuda.empty_cache()
        b1 = LayerTimer(d, layers, cfg.with_tokens(1), d.DYMOE_DECODE, ladder, device)
        subs["decode_b1"] = sub_line(b1, Ks, W, peaks)
        for name, (bits, lams) in PAPER_LADDERS.items():
            lad = d.make_ladder(bits, lams)
            desc = {"bits": bits, "lambdas": lams, "paper": "P:312 %s, r_mean = %.2f (D6)" % (
                name, (1 + lams[0]) / 2)}
            for B in (1, args.batch):
                t = LayerTimer(d, layers, cfg.with_tokens(B), d.DYMOE_DECODE, lad, device, ladder_desc=desc)
                subs["decode_b%d_ladder_%s" % (B, name.replace("/", "_"))] = sub_line(t, Ks, W, peaks, e2e=False)
        sweep = {}
        for b in (16, 8, 4, 2):
            forced = torch.full((cfg.M,), b, dtype=torch.uint8, device=device)
            t = LayerTimer(d, layers, cfg, d.DYMOE_DECODE, ladder, device, forced=forced,
                           ladder_desc={"forced_bits": b})
            t.run(min(K, 64), W)
            rf = t.roofline(peaks)
            sweep["int%d" % b if b != 16 else "bf16"] = {
                "w13_GBs": rf["achieved"], "w13_frac": rf["frac"], "w2_GBs": rf["w2_GBs"],
                "w2_frac": rf["w2_frac"], "tokens_per_s": t.T * t.res["K"] / (t.res["ms"] / 1e3)}
        subs["decode_width_sweep"] = dict(sweep, note="B = %d, every expert forced to one width "
                                          "(forced_bits), fractions of measured HBM" % cfg.T)
        res["sub_lines"] = subs
    res["quantize"] = measure_quantize(d, layers[0][1], cfg, peaks)
    res["next_rows"] = measure_extras(d, cfg, phase, device, peaks)
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(cfg, args, phase == d.DYMOE_PREFILL)
    return res


PAPER_LADDERS = {"4/2": ((4, 2), (0.5,)), "4/0": ((4, 0), (0.5,))}


def run_ep(args, rank, world, device):
    """N > 1: the expert-parallel layer through the C ABI (dymoe_moe_forward_ep): experts sharded
    in contiguous blocks over the ranks, every rank its own batch (weak scaling).  Both transports
    are timed -- the handle's own NCCL communicator (grouped send/recv of the (source, expert)
    chunks) and the peer-memory windows (fused dispatch / combine kernels, device flag barriers,
    no host synchronisation); the main line is the peer-memory path when its first steps run clean
    on every rank.  Decode also times the replicated-batch placement (strong scaling of one
    batch).  Timing: W warm-up steps, K steps between a barrier + synchronize on both sides,
    CUDA events on the launching stream, max over ranks."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200 import ep
    d.lib()
    torch.cuda.set_device(device)
    peaks = load_peaks()
    cfg, is_decode, wname = workload_cfg(args)
    T = cfg.T
    phase = d.DYMOE_DECODE if is_decode else d.DYMOE_PREFILL
    gloo = torch.distributed.get_backend() != "nccl"
    # gloo: the test hook of several ranks time-sharing ONE GPU -- NCCL refuses two ranks on one
    # device, so only the peer-memory transport (windows over CUDA IPC) runs there
    transports = d.DYMOE_EP_PEER if gloo else (d.DYMOE_EP_NCCL | d.DYMOE_EP_PEER)
    uid = None if gloo else ep.broadcast_unique_id()
    first, last = ep.owned_range(rank, cfg.M, world)
    layers = []
    setup_errors = {}
    for c in range(args.copies):
        ex = synthetic.expert_weights(cfg, 100 + c, device, experts=list(range(first, last)))
        ex = [{n: t.to(device) for n, t in e.items()} for e in ex]
        d.quantize_experts(ex, (8, 4, 2))
        try:
            L_ = ep.EPLayer(rank, world, cfg.M, cfg.k, cfg.hidden, cfg.ffn, T, ex,
                            transports=transports, nccl_uid=uid)
            ok = 1.0
        except d.DymoeError as err:   # e.g. no peer access between the GPUs: NCCL only
            setup_errors["peer"] = str(err)[:300]
            L_, ok = None, 0.0
        # every rank must agree on the transports (the window exchange is collective)
        if _max_over_ranks(1.0 - ok, device) > 0:
            if L_ is not None:
                L_.close()
            if gloo:
                raise SystemExit("expert-parallel handle creation failed: %s" % setup_errors)
            transports = d.DYMOE_EP_NCCL
            uid = ep.broadcast_unique_id()
            L_ = ep.EPLayer(rank, world, cfg.M, cfg.k, cfg.hidden, cfg.ffn, T, ex,
                            transports=transports, nccl_uid=uid)
        layers.append(L_)
        if gloo:
            opened = ep.connect_processes(layers[-1])
            layers[-1]._opened = opened
    torch.cuda.synchronize()
    n_inputs = 8
    inputs = []
    for i in range(n_inputs):
        x, lg, a = synthetic.layer_inputs(cfg, 1000 + i * 97 + rank, device)
        inputs.append((x.contiguous(), lg.contiguous(), a.contiguous()))
    ladder = d.make_ladder(LADDER_BITS, LADDER_LAMBDAS)
    K, W = args.steps, args.warmup
    ws = [L.workspace(T) for L in layers]
    out = torch.empty(T, cfg.hidden, dtype=torch.float32, device=device)

    def step(i, transport, placement=d.DYMOE_EP_ALL_TO_ALL, ev=None, x=None, lg=None, a=None, y=None):
        c = i % len(layers)
        if x is None:
            x, lg, a = inputs[i % n_inputs] if placement == d.DYMOE_EP_ALL_TO_ALL else rep_in
        layers[c].forward(x, lg, ladder, i % NUM_LAYERS, NUM_LAYERS, phase, transport=transport,
                          placement=placement, attn_mass=a, prof_events=ev,
                          ws=ws[c] if placement == d.DYMOE_EP_ALL_TO_ALL else wsr[c],
                          out=out if y is None else y)

    def status_all(placement=d.DYMOE_EP_ALL_TO_ALL):
        word = 0
        for c, L in enumerate(layers):
            word |= L.check_status(T, ws[c] if placement == d.DYMOE_EP_ALL_TO_ALL else wsr[c],
                                   placement=placement)[1]
        return int(_max_over_ranks(float(word), device))

    def census():
        """local algorithmic work of every distinct step: the rows this rank's experts receive
        (all ranks' per-expert counts, gathered untimed) at the widths the step assigned"""
        cen = {}
        for i in range(math.lcm(len(layers), NUM_LAYERS, n_inputs)):
            step(i, d.DYMOE_EP_NCCL if transports & d.DYMOE_EP_NCCL else d.DYMOE_EP_PEER)
            c = i % len(layers)
            v = layers[c].views(T, ws[c])
            cnt = torch.diff(v["expert_off"]).to(torch.int64)
            allc = _all_gather(cnt, device)
            rows = allc.sum(0).cpu().numpy()[first:last]
            bits = v["bits"].cpu().numpy()[first:last]
            sub = synthetic.MoEConfig("loc", M=last - first, k=1, hidden=cfg.hidden, ffn=cfg.ffn, T=T)
            off = np.concatenate([[0], np.cumsum(rows)])
            cen[(c, i % NUM_LAYERS, i % n_inputs)] = (algorithmic_bytes(sub, bits, off),
                                                      algorithmic_flops(sub, off, bits))
        return cen

    def timed(transport, placement=d.DYMOE_EP_ALL_TO_ALL):
        for i in range(W):
            step(i, transport, placement)
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
        for row in ev:
            for e_ in row:
                e_.record()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.distributed.barrier()
        torch.cuda.synchronize()
        prof = [i for i in range(K) if i % PROF_EVERY == 0]   # per-kernel events: a sample
        with ClockSampler(torch.cuda.current_device()) as clk:
            t0.record()
            for i in range(K):
                step(W + i, transport, placement, ev=ev[i] if i % PROF_EVERY == 0 else None)
            t1.record()
            torch.cuda.synchronize()
        torch.distributed.barrier()
        ms = _max_over_ranks(t0.elapsed_time(t1), device)
        w13 = sum(ev[i][0].elapsed_time(ev[i][1]) for i in prof)
        w2 = sum(ev[i][1].elapsed_time(ev[i][2]) for i in prof)
        return ms, w13, w2, clk.summary(), prof

    lines, errors = {}, {}
    cen = census()
    for name, tp in (("peer", d.DYMOE_EP_PEER), ("nccl", d.DYMOE_EP_NCCL)):
        if not (transports & tp):
            continue
        try:
            step(0, tp)                       # one step, then every rank's status, before timing
            torch.cuda.synchronize()
            if status_all():
                raise RuntimeError("status word after the first step")
            ms, w13, w2, clk, prof = timed(tp)
            st = status_all()
            steps = [((W + i) % len(layers), (W + i) % NUM_LAYERS, (W + i) % n_inputs) for i in prof]
            b13 = sum(cen[p][0][0] for p in steps)
            b2 = sum(cen[p][0][1] for p in steps)
            fl = sum(cen[p][1] for p in steps)
            lines[name] = {"value": T * K * world / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms / K,
                           "status": st, "clocks": clk, "w13_ms": w13, "w2_ms": w2, "b13": b13, "b2": b2,
                           "fl": fl, "K_prof": len(prof)}
        except Exception as ex:   # reported, never fatal for the other transport
            errors[name] = "%s: %s" % (type(ex).__name__, str(ex)[:300])
    main = "peer" if ("peer" in lines and lines["peer"]["status"] == 0 and args.ep_main != "nccl") \
        else ("nccl" if "nccl" in lines else None)
    if args.ep_main == "nccl" and "nccl" in lines:
        main = "nccl"
    if main is None:
        raise SystemExit("no expert-parallel transport ran: %s" % errors)
    L0 = lines[main]
    main_tp = d.DYMOE_EP_PEER if main == "peer" else d.DYMOE_EP_NCCL

    # ---------------- end-to-end through the main line: the rank's inputs from pinned host memory
    # and its output back to the host, every step, inside the timed region
    hx = [inp[0].cpu().pin_memory() for inp in inputs]
    hl = [inp[1].cpu().pin_memory() for inp in inputs]
    ha = [inp[2].cpu().pin_memory() for inp in inputs]
    dx, dl, da = (torch.empty_like(t) for t in inputs[0])
    hy = torch.empty(T, cfg.hidden, dtype=torch.float32).pin_memory()
    h2d = hx[0].numel() * 2 + hl[0].numel() * 4 + (ha[0].numel() * 4 if phase == d.DYMOE_PREFILL else 0)
    d2h = hy.numel() * 4
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.distributed.barrier()
    torch.cuda.synchronize()
    e0.record()
    for i in range(K):
        j = (W + i) % n_inputs
        dx.copy_(hx[j], non_blocking=True)
        dl.copy_(hl[j], non_blocking=True)
        if phase == d.DYMOE_PREFILL:
            da.copy_(ha[j], non_blocking=True)
        step(W + i, main_tp, x=dx, lg=dl, a=da)
        hy.copy_(out, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e2e = {"value": T * K * world / (_max_over_ranks(e0.elapsed_time(e1), device) / 1e3),
           "unit": "tokens/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---------------- decode, the same batch replicated on every rank (SURVEY §8e latency
    # variant): local experts, the partial outputs summed over the ranks; strong scaling
    rep = {}
    if phase == d.DYMOE_DECODE and T <= 64:
        rep_in = tuple(t.clone() for t in inputs[0])
        _broadcast(rep_in[0])
        _broadcast(rep_in[1])
        wsr = [L.workspace(T, placement=d.DYMOE_EP_REPLICATED) for L in layers]
        for name, tp in (("peer", d.DYMOE_EP_PEER), ("nccl", d.DYMOE_EP_NCCL)):
            if not (transports & tp):
                continue
            try:
                ms, _, _, clk, _ = timed(tp, d.DYMOE_EP_REPLICATED)
                rep[name] = {"value": T * K / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms / K,
                             "scaling": "strong", "global_batch": T,
                             "status": status_all(d.DYMOE_EP_REPLICATED)}
            except Exception as ex:
                rep[name] = {"error": "%s: %s" % (type(ex).__name__, str(ex)[:300])}

    # local FFN roofline of the main line (rank 0's experts: algorithmic bytes or flops / FFN time)
    ffn_ms = L0["w13_ms"] + L0["w2_ms"]
    if phase == d.DYMOE_DECODE:
        ach = L0["b13"] / max(L0["w13_ms"] / 1e3, 1e-12) / 1e9
        roof = {"bound": "hbm", "kernel": "k_decode_gemv<W13> on the rows rank 0 received",
                "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s", "frac": ach / peaks["hbm"],
                "traffic": None, "peak_src": peaks["src"],
                "ffn_w13_plus_w2_GBs": (L0["b13"] + L0["b2"]) / max(ffn_ms / 1e3, 1e-12) / 1e9,
                "ffn_share_of_step": ffn_ms / (L0["ms_per_step"] * L0["K_prof"]),
                "profiled_steps": L0["K_prof"], "prof_every": PROF_EVERY}
    else:
        ach = L0["fl"] / max(ffn_ms / 1e3, 1e-12) / 1e12
        pk = peaks["bf16_sus"] or peaks["bf16"]
        roof = {"bound": "tensor", "kernel": "k_prefill_gemm<W13> + <W2> on the rows rank 0 received",
                "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "traffic": None,
                "peak_src": peaks["src"] + " bf16 sustained",
                "ffn_share_of_step": ffn_ms / (L0["ms_per_step"] * L0["K_prof"]),
                "profiled_steps": L0["K_prof"], "prof_every": PROF_EVERY}
    for l in layers:
        for b in getattr(l, "_opened", []):
            d.dymoe_ep_window_close(b)
    torch.distributed.barrier()
    for l in layers:
        l.close()
    if rank != 0:
        return None
    pub = lambda v: {k: v[k] for k in ("value", "unit", "ms_per_step", "status")}
    return {"metric": METRIC, "value": L0["value"], "unit": "tokens/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": L0["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 x int8/int4/int2 (fp32 accum)",
            "data": "synthetic (seeded random-init Mixtral-8x7B-shaped experts, Zipf-skewed router logits)",
            "config": {"workload": wname, "hidden": cfg.hidden, "ffn": cfg.ffn,
                       "experts": cfg.M, "top_k": cfg.k, "tokens_per_step_per_rank": T,
                       "global_batch": T * world,
                       "ladder": {"bits": LADDER_BITS, "lambdas": LADDER_LAMBDAS},
                       "schedule": "layer l = step mod 32 of a 32-layer depth schedule",
                       "weight_copies": args.copies, "l2": "inputs larger than L2 (rotating weight copies)",
                       "parallelism": "ep%d: experts sharded, dymoe_moe_forward_ep over %s" % (
                           world, "peer-memory windows (fused dispatch/combine kernels)" if main == "peer"
                           else "the library's NCCL communicator (grouped send/recv)")},
            "roofline": roof, "clocks": L0["clocks"], "e2e": e2e,
            # libdymoe launches per step and rank (peer: route, score, publish, barrier, reduce,
            # assign, permute, dispatch, barrier, active list, W13, W2, reduce/zero, barrier,
            # combine; NCCL: route, score, assign, permute, counts, gather, active, W13, W2,
            # reduce/zero, combine -- NCCL's own kernels not counted)
            "gpu_launches": (15 if main == "peer" else 11) * K,
            "ep_path": main, "ep_transports": {k: pub(v) for k, v in lines.items()},
            "ep_errors": dict(errors, **setup_errors) or None, "ep_replicated_decode": rep or None}


def _all_gather(t, device):
    ws = torch.distributed.get_world_size()
    if torch.distributed.get_backend() == "nccl":
        out = [torch.empty_like(t) for _ in range(ws)]
        torch.distributed.all_gather(out, t)
    else:
        c = t.cpu()
        out = [torch.empty_like(c) for _ in range(ws)]
        torch.distributed.all_gather(out, c)
    return torch.stack(out)


def _max_over_ranks(v, device):
    """max of a host float over the ranks (CUDA tensor for NCCL, CPU tensor for gloo)."""
    dev = device if torch.distributed.get_backend() == "nccl" else torch.device("cpu")
    tt = torch.tensor([v], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    return float(tt.item())


def _broadcast(t):
    if torch.distributed.get_backend() == "nccl":
        torch.distributed.broadcast(t, 0)
    else:
        c = t.cpu()
        torch.distributed.broadcast(c, 0)
        t.copy_(c)


def load_traffic(kernel_key):
    """dram read+write bytes of the dominant kernel from the committed ncu --set full capture
    (profiles/traffic.json, written from the committed ncu summaries, profiles/r02_final_ncu_*.md), with the algorithmic work of
    the same captured launch so the two can be compared."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    return j.get(kernel_key)


def measure_extras(d, cfg, phase, device, peaks, reps=10):
    """SURVEY §8f rows built beside the path, timed alone (CUDA events): the look-ahead expert
    predictor (Eqs. 6-8) on this workload's tokens, and the causal attention mass (f3) for a
    Mixtral-shaped attention (H = 32, d = 128) over this workload's tokens (prefill)."""
    out = {}
    T = cfg.T
    g = torch.Generator(device=device).manual_seed(11)
    h = torch.randn(T, cfg.hidden, generator=g, device=device).to(torch.bfloat16)
    wg = (torch.randn(cfg.M, cfg.hidden, generator=g, device=device) / cfg.hidden ** 0.5).to(torch.bfloat16)
    nbytes = d.lib().dymoe_predict_ws_bytes(T, cfg.M, cfg.k)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    ex = torch.empty(cfg.M, dtype=torch.int32, device=device)
    pr = torch.empty(cfg.M, dtype=torch.float32, device=device)
    n = torch.empty(1, dtype=torch.int32, device=device)
    st = torch.cuda.current_stream()

    def predict():
        d._check(d.lib().dymoe_predict_next(phase, d._p(d._u16(h)), d._p(d._u16(wg)), T, cfg.hidden,
                                            cfg.M, cfg.k, 2, d._p(ws), nbytes, d._p(ex), d._p(pr),
                                            d._p(n), None, d._stream(st)))

    def timed(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    us = timed(predict)
    out["predict_next"] = {"us": us, "GB/s": (T * cfg.hidden * 2) / (us * 1e-6) / 1e9,
                           "note": "Eq. 6 gate product + Eq. 7/8 selection, h [T][Hd] read once"}
    if phase == d.DYMOE_PREFILL:
        H = 32
        q = torch.randn(H, T, 128, generator=g, device=device).to(torch.bfloat16)
        k = torch.randn(H, T, 128, generator=g, device=device).to(torch.bfloat16)
        us = timed(lambda: d.dymoe_attention_mass(q, k))
        fl = 2 * 2 * T * T * 128 * H / 2
        tf = fl / (us * 1e-6) / 1e12
        out["attention_mass"] = {"us": us, "TFLOP/s": tf, "frac_bf16_burst": tf / peaks["bf16"],
                                 "H": H, "d": 128, "T": T,
                                 "note": "two causal Q.K^T passes on tcgen05 (row stats, column sums "
                                         "of P from TMEM), 2 x 2 T^2 d H / 2 flops; timed alone"}
    return out


def measure_quantize(d, experts, cfg, peaks, reps=5):
    out = {}
    ex = experts[0]
    for b in (8, 4, 2):
        jobs = [(ex[n], b, ex["q%d" % b][n]) for n in ("w1", "w3", "w2")]
        d.dymoe_quantize_batched(jobs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            d.dymoe_quantize_batched(jobs)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / reps / 1e3
        nbytes = 3 * cfg.hidden * cfg.ffn * (2 + bytes_per_weight(b))
        gbs = nbytes / s / 1e9
        out["int%d" % b] = {"GB/s": gbs, "frac": gbs / peaks["hbm"], "us": s * 1e6,
                            "bytes": nbytes}
    out["note"] = "one Mixtral expert (W1, W3, W2) per launch; 352 MB bf16 read, > L2 per rep"
    return out


# =============================================================================================
_CPU_INPUTS = {}


def cpu_baseline(cfg, args, prefill, frac=8):
    """The oracle as it stands, on this host's cores, on a bounded sample of one step."""
    from oracle import moe as o_moe, route as o_route, importance as o_imp, schedule as o_sched
    cores = len(os.sched_getaffinity(0))
    key = (cfg, prefill)
    if key not in _CPU_INPUTS:   # input generation is not part of the timed sample
        _CPU_INPUTS[key] = (synthetic.layer_inputs(cfg, 1000),
                            synthetic.expert_weights(cfg, 100, experts=[0]))
    (x, lg, a), ex = _CPU_INPUTS[key]
    t0 = time.perf_counter()
    idx, w, p = o_route.route(lg.numpy(), cfg.k)
    if prefill:
        I, _, _ = o_imp.score_prefill(a.numpy(), idx, cfg.M)
    else:
        I = o_imp.decode_importance(lg.numpy(), p)
    bits, _ = o_sched.assign_bits(I, 16, NUM_LAYERS, o_sched.Ladder(LADDER_BITS, LADDER_LAMBDAS), cfg.k)
    perm = o_moe.permute(idx, bits, cfg.M)
    t_ctrl = time.perf_counter() - t0
    # FFN sample: 1/frac of expert 0's rows (W1/W3 rows and the matching W2 columns) at its width
    e0 = ex[0]
    Fs = max(128, cfg.ffn // frac // 128 * 128)   # whole quantization groups of W2's K
    frac = cfg.ffn / Fs
    sub = {"w1": e0["w1"][:Fs].float().numpy(), "w3": e0["w3"][:Fs].float().numpy(),
           "w2": e0["w2"][:, :Fs].contiguous().float().numpy()}
    b = int(bits[0]) or 4
    n_rows = max(int(perm["expert_off"][1] - perm["expert_off"][0]), 1)
    t1 = time.perf_counter()
    W1, W3, W2 = o_moe.expert_weights(sub, b)
    rows = perm["perm_token"][perm["expert_off"][0]:perm["expert_off"][1]]
    xr = x.float().numpy()[rows if len(rows) else [0]].astype(np.float64)
    o_moe.ffn(xr, W1, W3, W2)
    t_ffn = (time.perf_counter() - t1) * frac
    n_active = int((np.diff(perm["expert_off"]) > 0).sum())
    step_s = t_ctrl + t_ffn * n_active
    return {"value": cfg.T / step_s, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": "route+score+assign+permute for all %d tokens; FFN of 1/%g of one expert "
                      "(Int%d, %d rows) scaled x%g and x%d active experts" % (cfg.T, frac, b, n_rows, frac, n_active),
            "blas_threads": torch.get_num_threads(), "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """Reference arm: the CPU oracle on the same workload, bounded sample per step."""
    cfg, is_decode, wname = workload_cfg(args)
    T = cfg.T
    prefill = not is_decode
    for _ in range(args.warmup):
        cpu_baseline(cfg, args, prefill, frac=64)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(cfg, args, prefill, frac=64))
    wall = time.perf_counter() - t0
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[0])
    cb["value"] = v
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)",
            "data": "synthetic", "config": {"workload": wname, "tokens_per_step": T},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_stack(args, device):
    """SURVEY §8d C5 (BASELINE.json configs[4]) on one GPU: a 32-layer Mixtral-8x7B-shaped stack
    on the bf16 residual stream (paper_2603_19172_b200.stack.MoEStack: RMSNorm -> router -> MoE ->
    residual add per layer), every layer its own random
    experts (packed Int8/Int4/Int2 resident, bf16 masters dropped after quantization: 84 GB) and
    its own router, depth-adaptive bits.  A step = one pass of the whole stack for `batch` decode
    tokens (or `tokens` prefill tokens).  value = tokens through all 32 layers per second."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200.stack import MoEStack
    d.lib()
    torch.cuda.set_device(device)
    peaks = load_peaks()
    prefill = args.workload == "stack_prefill"
    T = args.tokens if prefill else args.batch
    cfg = synthetic.CONFIGS["stack"].with_tokens(T)
    L = cfg.layers
    phase = d.DYMOE_PREFILL if prefill else d.DYMOE_DECODE
    layers, gates = [], []
    for l in range(L):
        ex = [{n: t for n, t in e.items()} for e in synthetic.expert_weights(cfg, 3000 + l, device)]
        d.quantize_experts(ex, (8, 4, 2))
        torch.cuda.synchronize()
        for e in ex:          # the ladder has no BF16 tier: keep only the packed widths
            for n in ("w1", "w3", "w2"):
                del e[n]
        layers.append(ex)
        gates.append(synthetic.stack_gate(cfg, l, 7, device))
    torch.cuda.empty_cache()
    st = MoEStack(layers, gates, cfg.k, cfg.hidden, cfg.ffn)
    x = synthetic.hidden_states(cfg, 8, device)
    attn = [synthetic.attention_mass(cfg, 400 + l, device) for l in range(L)] if prefill else None
    ladder = d.make_ladder(LADDER_BITS, LADDER_LAMBDAS)
    ws = st.workspace(T, device)
    bufs = (torch.empty_like(x), torch.empty_like(x), torch.empty_like(x))
    logits = torch.empty(T, cfg.M, dtype=torch.float32, device=device)
    # census of one pass (bits and loads are data-dependent per layer)
    _, tr = st.forward(x, ladder, phase, attn, ws=ws, bufs=bufs, logits=logits, trace=True)
    b_tot = fl_tot = 0.0
    widths = {}
    for l in range(L):
        bits = tr[l][3].cpu().numpy()
        lgl = tr[l][2]
        r_idx = torch.topk(lgl, cfg.k, dim=1).indices.cpu().numpy()   # loads only (census)
        off = np.zeros(cfg.M + 1, np.int64)
        for e in range(cfg.M):
            off[e + 1] = off[e] + int((r_idx == e).sum()) * int(bits[e] != 0)
        b13, b2 = algorithmic_bytes(cfg, bits, off)
        b_tot += b13 + b2
        fl_tot += algorithmic_flops(cfg, off, bits)
        for b in bits.tolist():
            widths[b] = widths.get(b, 0) + 1
    del tr
    stream = torch.cuda.current_stream()

    def one_step():
        st.forward(x, ladder, phase, attn, ws=ws, bufs=bufs, logits=logits)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    # the whole 32-layer pass (6-10 launches per layer, no host synchronisation inside) captured
    # once as a CUDA graph and replayed: launch gaps and host marshalling leave the timed loop
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                one_step()
        stream.wait_stream(side)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    K = args.steps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0.record(stream)
        for _ in range(K):
            if graph is not None:
                graph.replay()
            else:
                one_step()
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    # e2e: x from pinned host memory in, the final stream out, every step
    hx = x.cpu().pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    dx = torch.empty_like(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(K):
        dx.copy_(hx, non_blocking=True)
        y, _ = st.forward(dx, ladder, phase, attn, ws=ws, bufs=bufs, logits=logits)
        hy.copy_(y, non_blocking=True)
    # (e2e runs the public API call by call, no graph: what a caller of MoEStack.forward gets)
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    step_s = ms / K / 1e3
    if prefill:
        ach = fl_tot / step_s / 1e12
        pk = peaks["bf16_sus"] or peaks["bf16"]
        roof = {"bound": "tensor", "kernel": "whole stack (32 x (rmsnorm, gate, front, tcgen05 W13/W2 GEMMs, combine))",
                "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "traffic": None,
                "peak_src": peaks["src"] + " bf16 sustained", "algorithmic_flops_per_step": fl_tot}
    else:
        ach = b_tot / step_s / 1e9
        roof = {"bound": "hbm", "kernel": "whole stack (32 x (rmsnorm, gate, front, W13/W2 GEMVs, combine))",
                "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s", "frac": ach / peaks["hbm"],
                "traffic": None, "peak_src": peaks["src"], "algorithmic_bytes_per_step": b_tot}
    # rmsnorm, gate, (decode: fused front | prefill: route, score, assign, permute, gather), W13,
    # W2, combine
    per_layer = 6 if not prefill else 10
    return {"metric": METRIC, "value": T * K / (ms / 1e3), "unit": "tokens/s", "n_gpus": 1, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 x int8/int4/int2 (fp32 accum)",
            "data": "synthetic (seeded random-init Mixtral-8x7B-shaped experts and routers per layer)",
            "config": {"workload": "mixtral_stack32_%s" % ("prefill" if prefill else "decode"),
                       "layers": L, "hidden": cfg.hidden, "ffn": cfg.ffn, "experts": cfg.M, "top_k": cfg.k,
                       "tokens_per_step": T, "ladder": {"bits": LADDER_BITS, "lambdas": LADDER_LAMBDAS},
                       "resident_packed_GB": round(torch.cuda.memory_allocated() / 1e9, 1),
                       "widths_assigned": {str(k): v for k, v in sorted(widths.items())},
                       "l2": "inputs larger than L2 (32 distinct layers, 84 GB of packed weights)",
                       "parallelism": "single GPU"},
            "ms_per_layer": ms / K / L, "cuda_graph": graph is not None, "roofline": roof, "clocks": clk.summary(),
            "e2e": {"value": T * K / (e_ms / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(hx.numel() * 2), "d2h_bytes_per_step": int(hy.numel() * 2)},
            "gpu_launches": per_layer * L * K}


def run_stack_ep(args, rank, world, device):
    """SURVEY §8d C5 / BASELINE.json configs[4] as named: the 32-layer Mixtral-8x7B-shaped stack
    expert-parallel over the ranks (paper_2603_19172_b200.stack.EPStack: per layer RMSNorm and
    router on the rank's own tokens, then dymoe_moe_forward_ep -- global importance, exchange,
    owners' fused-dequant FFN, combine with the residual).  Each rank holds its block of every
    layer's experts (packed widths only) and brings its own batch (weak scaling).  value = tokens
    of all ranks through all 32 layers per second (max over ranks)."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200 import ep
    from paper_2603_19172_b200.stack import EPStack
    d.lib()
    torch.cuda.set_device(device)
    peaks = load_peaks()
    prefill = args.workload == "stack_prefill"
    T = args.tokens if prefill else args.batch
    cfg = synthetic.CONFIGS["stack"].with_tokens(T)
    L = cfg.layers
    phase = d.DYMOE_PREFILL if prefill else d.DYMOE_DECODE
    gloo = torch.distributed.get_backend() != "nccl"
    transports = d.DYMOE_EP_PEER if gloo else (d.DYMOE_EP_NCCL | d.DYMOE_EP_PEER)
    uid = None if gloo else ep.broadcast_unique_id()
    first, last = ep.owned_range(rank, cfg.M, world)
    local = []
    for l in range(L):
        ex = synthetic.expert_weights(cfg, 3000 + l, device, experts=list(range(first, last)))
        ex = [{n: t for n, t in e.items()} for e in ex]
        d.quantize_experts(ex, (8, 4, 2))
        torch.cuda.synchronize()
        for e in ex:          # the ladder has no BF16 tier: keep only the packed widths
            for n in ("w1", "w3", "w2"):
                del e[n]
        local.append(ex)
    torch.cuda.empty_cache()
    h = ep.EPLayer(rank, world, cfg.M, cfg.k, cfg.hidden, cfg.ffn, T, local[0],
                   transports=transports, nccl_uid=uid)
    opened = ep.connect_processes(h) if gloo else []
    gates = [synthetic.stack_gate(cfg, l, 7, device) for l in range(L)]
    st = EPStack(h, local, gates)
    x = synthetic.hidden_states(cfg, 8 + rank, device)
    attn = [synthetic.attention_mass(cfg, 400 + l, device) for l in range(L)] if prefill else None
    ladder = d.make_ladder(LADDER_BITS, LADDER_LAMBDAS)
    ws = h.workspace(T)
    bufs = (torch.empty_like(x), torch.empty_like(x), torch.empty_like(x))
    logits = torch.empty(T, cfg.M, dtype=torch.float32, device=device)
    K, W = args.steps, args.warmup
    lines = {}
    for name, tp in (("peer", d.DYMOE_EP_PEER), ("nccl", d.DYMOE_EP_NCCL)):
        if not (transports & tp):
            continue
        for _ in range(W):
            st.forward(x, ladder, phase, tp, attn, ws=ws, bufs=bufs, logits=logits)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            t0.record()
            for _ in range(K):
                st.forward(x, ladder, phase, tp, attn, ws=ws, bufs=bufs, logits=logits)
            t1.record()
            torch.cuda.synchronize()
        torch.distributed.barrier()
        ms = _max_over_ranks(t0.elapsed_time(t1), device)
        word = int(_max_over_ranks(float(h.check_status(T, ws)[1]), device))
        lines[name] = {"value": T * world * K / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms / K,
                       "status": word, "clocks": clk.summary()}
    main = "peer" if "peer" in lines and lines["peer"]["status"] == 0 else "nccl"
    tp_main = d.DYMOE_EP_PEER if main == "peer" else d.DYMOE_EP_NCCL
    L0 = lines[main]
    # e2e: the rank's x from pinned host memory in, its final stream out, every pass
    hx = x.cpu().pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    dx = torch.empty_like(x)
    torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        dx.copy_(hx, non_blocking=True)
        y, _ = st.forward(dx, ladder, phase, tp_main, attn, ws=ws, bufs=bufs, logits=logits)
        hy.copy_(y, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    e_ms = _max_over_ranks(e0.elapsed_time(e1), device)
    torch.distributed.barrier()
    ep.disconnect(opened)
    h.close()
    if rank != 0:
        return None
    return {"metric": METRIC, "value": L0["value"], "unit": "tokens/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": L0["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 x int8/int4/int2 (fp32 accum)",
            "data": "synthetic (seeded random-init Mixtral-8x7B-shaped experts and routers per layer)",
            "config": {"workload": "mixtral_stack32_%s" % ("prefill" if prefill else "decode"),
                       "layers": L, "hidden": cfg.hidden, "ffn": cfg.ffn, "experts": cfg.M, "top_k": cfg.k,
                       "tokens_per_step_per_rank": T, "global_batch": T * world,
                       "ladder": {"bits": LADDER_BITS, "lambdas": LADDER_LAMBDAS},
                       "l2": "inputs larger than L2 (32 distinct layers of packed weights)",
                       "parallelism": "ep%d: every layer's experts sharded, dymoe_moe_forward_ep over %s" % (
                           world, "peer-memory windows" if main == "peer" else "the library's NCCL communicator")},
            "ms_per_layer": L0["ms_per_step"] / L, "roofline": None, "clocks": L0["clocks"],
            "e2e": {"value": T * world * K / (e_ms / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(hx.numel() * 2), "d2h_bytes_per_step": int(hy.numel() * 2)},
            "gpu_launches": (17 if main == "peer" else 13) * L * K,
            "ep_path": main, "ep_transports": {k: {kk: v[kk] for kk in ("value", "ms_per_step", "status")}
                                               for k, v in lines.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="decode",
                    choices=["decode", "prefill", "finegrained", "finegrained_decode", "stack",
                             "stack_prefill"],
                    help="decode / prefill: one Mixtral layer (configs[1] / [2]); finegrained / "
                         "finegrained_decode: the 64-expert top-6 layer of configs[3]; stack / "
                         "stack_prefill: the 32-layer stack of configs[4] on one GPU")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--prof-every", type=int, default=17,
                    help="per-kernel CUDA events on every n-th timed step only: the kernel "
                         "roofline comes from those steps; each event is a node in the step's "
                         "CUDA graph and, on every step, cost the decode step ~14 us of its 214")
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--main-only", action="store_true",
                    help="decode workload: skip the sub-lines (prefill, B = 1, the paper's ladders, "
                         "the per-width sweep) that the default line carries")
    ap.add_argument("--no-graph", action="store_true", help="time the steps call by call instead "
                    "of replaying their CUDA graph (single-GPU decode / prefill / stack workloads)")
    ap.add_argument("--ep-main", default="auto", choices=["auto", "nccl", "peer"],
                    help="N > 1: the main line's transport (auto: the peer-memory windows when they "
                         "run clean on every rank, else the library's NCCL communicator)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test hook for several ranks sharing one GPU (collectives staged "
                         "through host memory); never used for reported numbers")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    global PROF_EVERY
    PROF_EVERY = max(1, args.prof_every)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched as `python bench.py --gpus N`: become the launcher of N ranks (one process per
        # GPU, torch.distributed.run on 127.0.0.1), relay their output and exit code
        import socket
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit("bench.py: WORLD_SIZE=%d but --gpus %d" % (world, args.gpus))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)))
        return
    if world > 1:
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group("gloo")
    if args.workload.startswith("stack"):
        if world > 1:
            res = run_stack_ep(args, rank, world, torch.device("cuda", local))
        else:
            res = run_stack(args, torch.device("cuda", local))
    elif world > 1:
        res = run_ep(args, rank, world, torch.device("cuda", local))
    else:
        res = run_ours(args, rank, world, torch.device("cuda", local))
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
