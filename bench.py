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


def step_inputs(cfg, n, device):
    out = []
    for i in range(n):
        x, lg, a = synthetic.layer_inputs(cfg, 1000 + i, device)
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


def run_ours(args, rank, world, device):
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    torch.cuda.set_device(device)
    peaks = load_peaks()
    cfg, is_decode, wname = workload_cfg(args)
    T = cfg.T
    phase = d.DYMOE_DECODE if is_decode else d.DYMOE_PREFILL
    layers = build_layer_copies(d, cfg, args.copies, device)
    n_inputs = 8
    inputs = step_inputs(cfg, n_inputs, device)
    ladder = d.make_ladder(LADDER_BITS, LADDER_LAMBDAS)
    ws = [L.workspace(T, device) for L, _ in layers]
    out = torch.empty(T, cfg.hidden, dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream()

    def plan(i):
        return i % len(layers), i % NUM_LAYERS, i % n_inputs

    events = None
    ffn_mode = d.DYMOE_FFN_PREFILL_TS if (phase == d.DYMOE_PREFILL and args.prefill_kernel == "ts") else -1

    def one_step(i, ev=None):
        c, l, j = plan(i)
        L = layers[c][0]
        x, lg, a = inputs[j]
        L.forward(x, lg, ladder, l, NUM_LAYERS, phase=phase, attn_mass=a, ws=ws[c], out=out,
                  prof_events=ev, ffn_mode=ffn_mode)

    # census: algorithmic bytes / flops of every distinct step (bits are data-dependent)
    census = {}
    period = math.lcm(len(layers), NUM_LAYERS, n_inputs)
    for i in range(period):
        one_step(i)
        c = plan(i)[0]
        v = layers[c][0].views(T, ws[c])
        bits = v["bits"].cpu().numpy()
        off = v["expert_off"].cpu().numpy()
        census[plan(i)] = (algorithmic_bytes(cfg, bits, off), algorithmic_flops(cfg, off, bits),
                           int((np.diff(off) > 0).sum()))
        rc, word = layers[c][0].check_status(T, ws[c])
        assert rc == 0, "device status word %x" % word
    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()

    # ---------------- timed region (device events, max over ranks)
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    for row in ev:
        for e_ in row:
            e_.record(stream)   # creates the CUDA event so its handle can be passed down
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the K steps (4 launches each in decode, no host synchronisation inside dymoe_moe_forward)
    # are captured once as a CUDA graph -- per-kernel events included -- and replayed in the timed
    # region, as a serving loop would: launch gaps and host-side marshalling leave the step
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=device)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                for i in range(K):
                    one_step(args.warmup + i, ev[i])
        stream.wait_stream(side)
        graph.replay()          # one untimed replay (the warm-up steps above ran call by call)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(K):
                one_step(args.warmup + i, ev[i])
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=device)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / K
    tokens = T * K * world
    value = tokens / (ms / 1e3)

    w13_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in range(K)]
    w2_ms = [ev[i][1].elapsed_time(ev[i][2]) for i in range(K)]
    b13 = sum(census[plan(args.warmup + i)][0][0] for i in range(K))
    b2 = sum(census[plan(args.warmup + i)][0][1] for i in range(K))
    fl = sum(census[plan(args.warmup + i)][1] for i in range(K))
    ffn_ms = sum(w13_ms) + sum(w2_ms)
    achieved_w13 = b13 / (sum(w13_ms) / 1e3) / 1e9
    achieved_ffn = (b13 + b2) / (ffn_ms / 1e3) / 1e9
    # the committed ncu capture is of the Mixtral layer's kernels
    tr = load_traffic("k_decode_gemv<W13>" if phase == d.DYMOE_DECODE else "k_prefill_gemm<W13>") \
        if wname.startswith("mixtral") else None
    traffic = tr["traffic"] if tr else None

    # ---------------- end-to-end through the public API with host buffers
    e2e = None
    if rank == 0 or world > 1:
        hx = [inp[0].cpu().pin_memory() for inp in inputs]
        hl = [inp[1].cpu().pin_memory() for inp in inputs]
        ha = [inp[2].cpu().pin_memory() for inp in inputs]
        # double-buffered device inputs / outputs; the copies run on a side stream so that step
        # i+1's inputs and step i-1's output move while step i computes (what a serving loop does)
        dbuf = [tuple(torch.empty_like(t) for t in inputs[0]) for _ in range(2)]
        obuf = [torch.empty(T, cfg.hidden, dtype=torch.float32, device=device) for _ in range(2)]
        hy = [torch.empty(T, cfg.hidden, dtype=torch.float32).pin_memory() for _ in range(2)]
        h2d = hx[0].numel() * 2 + hl[0].numel() * 4 + (ha[0].numel() * 4 if phase == d.DYMOE_PREFILL else 0)
        d2h = hy[0].numel() * 4
        cstream = torch.cuda.Stream(device=device)
        in_ready = [torch.cuda.Event() for _ in range(2)]
        out_ready = [torch.cuda.Event() for _ in range(2)]
        buf_free = [torch.cuda.Event() for _ in range(2)]
        out_free = [torch.cuda.Event() for _ in range(2)]

        def stage_in(i):
            _, _, j = plan(args.warmup + i)
            b = i & 1
            with torch.cuda.stream(cstream):
                cstream.wait_event(buf_free[b])
                dbuf[b][0].copy_(hx[j], non_blocking=True)
                dbuf[b][1].copy_(hl[j], non_blocking=True)
                if phase == d.DYMOE_PREFILL:
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
            c, l, j = plan(args.warmup + i)
            b = i & 1
            if i + 1 < K:
                stage_in(i + 1)
            stream.wait_event(in_ready[b])
            stream.wait_event(out_free[b])          # step i-2's output has left the device
            dx, dl, da = dbuf[b]
            layers[c][0].forward(dx, dl, ladder, l, NUM_LAYERS, phase=phase, attn_mass=da,
                                 ws=ws[c], out=obuf[b])
            buf_free[b].record(stream)
            out_ready[b].record(stream)
            with torch.cuda.stream(cstream):
                cstream.wait_event(out_ready[b])
                hy[b].copy_(obuf[b], non_blocking=True)
                out_free[b].record(cstream)
        e1.record(cstream)                            # after the last output copy
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([e_ms], device=device)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(tt.item())
        e2e = {"value": T * K * world / (e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---------------- quantize kernel (row a4), alone: one Mixtral expert per width
    quant = measure_quantize(d, layers[0][1], cfg, peaks)
    extras = measure_extras(d, cfg, phase, device, peaks)

    if phase == d.DYMOE_DECODE:
        # dominant kernel: the W1/W3 fused-dequant SwiGLU GEMV (HBM-bound); per launch the
        # algorithmic bytes are the packed W1+W3 bytes of the active experts (+ x, h)
        roofline = {"bound": "hbm", "kernel": "k_decode_gemv<W13> (fused-dequant SwiGLU GEMV)",
                    "achieved": achieved_w13, "peak": peaks["hbm"], "unit": "GB/s",
                    "frac": achieved_w13 / peaks["hbm"], "traffic": traffic,
                    "traffic_capture": tr, "peak_src": peaks["src"], "frac_of_8TBs": achieved_w13 / 8000.0,
                    "ffn_w13_plus_w2_GBs": achieved_ffn,
                    "ffn_share_of_step": ffn_ms / ms if world == 1 else None,
                    "algorithmic_bytes_per_step": (b13 + b2) / K}
    else:
        # dominant kernel: the tcgen05 fused-dequant grouped GEMMs (tensor-bound); algorithmic
        # flops per step = 6 * Hd * F per executed (token, expert) pair
        tfl = fl / (ffn_ms / 1e3) / 1e12
        tfl13 = (fl * 2 / 3) / (sum(w13_ms) / 1e3) / 1e12
        pk = peaks["bf16_sus"] or peaks["bf16"]
        roofline = {"bound": "tensor", "kernel": "k_prefill_gemm<W13> + <W2> (tcgen05 fused-dequant grouped GEMM)",
                    "achieved": tfl, "peak": pk, "unit": "TFLOP/s", "frac": tfl / pk,
                    "traffic": traffic, "traffic_capture": tr, "peak_src": peaks["src"] + " bf16 sustained",
                    "frac_of_2250": tfl / 2250.0, "w13_tflops": tfl13,
                    "w2_tflops": (fl / 3) / (sum(w2_ms) / 1e3) / 1e12,
                    "ffn_share_of_step": ffn_ms / ms if world == 1 else None,
                    "algorithmic_flops_per_step": fl / K, "hbm_GBs_ffn": achieved_ffn}
    res = None
    if rank == 0:
        # decode: fused front (route+score+assign+permute), W13, W2, combine; prefill: route, score,
        # assign, permute, gather into expert order, W13, W2, combine
        launches_per_step = 4 if phase == d.DYMOE_DECODE else 8
        res = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 x int8/int4/int2 (fp32 accum)",
            "data": "synthetic (seeded random-init Mixtral-8x7B-shaped experts, Zipf-skewed router logits)",
            "config": {"workload": wname, "hidden": cfg.hidden, "ffn": cfg.ffn,
                       "experts": cfg.M, "top_k": cfg.k, "tokens_per_step": T,
                       "ladder": {"bits": LADDER_BITS, "lambdas": LADDER_LAMBDAS},
                       "schedule": "layer l = step mod 32 of a 32-layer depth schedule",
                       "weight_copies": args.copies,
                       "l2": "inputs larger than L2: %d rotating weight copies of %.1f GB each (L2 126 MB)" % (
                           args.copies, cfg.M * 3 * cfg.hidden * cfg.ffn * sum(
                               bytes_per_weight(b) for b in (16, 8, 4, 2)) / 1e9),
                       "parallelism": "replicas" if world > 1 else "single GPU"},
            "roofline": roofline,
            "clocks": clk.summary(),
            "e2e": e2e,
            "gpu_launches": launches_per_step * K,
            "cuda_graph": graph is not None,
            "prefill_kernel": args.prefill_kernel if phase == d.DYMOE_PREFILL else None,
            "quantize": quant,
            "next_rows": extras,
            "tensor_tflops_ffn": fl / (ffn_ms / 1e3) / 1e12,
        }
        if not args.no_cpu_baseline and world == 1:
            res["cpu_baseline"] = cpu_baseline(cfg, args, phase == d.DYMOE_PREFILL)
    return res


def run_ep(args, rank, world, device):
    """N > 1: expert-parallel layer (experts sharded in contiguous blocks over the ranks, NCCL
    all-to-all dispatch/combine via paper_2603_19172_b200.ep); every rank brings its own batch
    (weak scaling).  Timed exactly like the single-GPU run; max over ranks."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200 import ep
    d.lib()
    torch.cuda.set_device(device)
    peaks = load_peaks()
    cfg, is_decode, wname = workload_cfg(args)
    T = cfg.T
    phase = d.DYMOE_DECODE if is_decode else d.DYMOE_PREFILL
    comm = ep.TorchComm(stage_cpu=torch.distributed.get_backend() != "nccl")

    class TimedOps(ep.CudaOps):
        """CudaOps recording CUDA events around the local expert FFN (roofline numerator)."""

        def __init__(self):
            super().__init__()
            self.events, self.rows = [], []

        def expert_ffn(self, layer, x_rows, bits, expert_off, perm_token, mode):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            y = super().expert_ffn(layer, x_rows, bits, expert_off, perm_token, mode)
            e1.record()
            self.events.append((e0, e1, bits, expert_off))
            return y

    ops = TimedOps()
    first, last = ep.owned_range(rank, cfg.M, world)
    shards = []
    for c in range(args.copies):
        ex = [{n: t.to(device) for n, t in e.items()}
              for e in synthetic.expert_weights(cfg, 100 + c, device, experts=list(range(first, last)))]
        ex = ex[first:last] if len(ex) > last - first else ex
        d.quantize_experts(ex, (8, 4, 2))
        shards.append(ep.EPMoELayer(comm, ops, ex, cfg.M, cfg.k, cfg.hidden, cfg.ffn,
                                    make_local_layer=lambda e_: d.MoELayer(e_, 1, cfg.hidden, cfg.ffn)))
    n_inputs = 8
    inputs = []
    for i in range(n_inputs):
        x, lg, a = synthetic.layer_inputs(cfg, 1000 + i * 97 + rank, device)
        inputs.append((x.contiguous(), lg.contiguous(), a.contiguous()))
    ladder = d.make_ladder(LADDER_BITS, LADDER_LAMBDAS)

    def one_step(i):
        x, lg, a = inputs[i % n_inputs]
        return shards[i % len(shards)].forward(x, lg, ladder, i % NUM_LAYERS, NUM_LAYERS, phase,
                                               attn_mass=a)

    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()
    K = args.steps
    ops.events.clear()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0.record()
        for i in range(K):
            one_step(args.warmup + i)
        t1.record()
        torch.cuda.synchronize()
    torch.distributed.barrier()
    ms = t0.elapsed_time(t1)
    ms = _max_over_ranks(ms, device)
    value = T * K * world / (ms / 1e3)
    ffn_events = list(ops.events)

    # ---------------- the same weak-scaling steps with dispatch / combine over peer memory
    # (forward_p2p: fused gather+store and pull+combine kernels, flag barriers).  It
    # is the main line when it runs clean on every rank; the NCCL all-to-all line is kept beside it
    p2p, win = None, None
    nccl_ms = ms
    try:
        gloo = torch.distributed.get_backend() != "nccl"
        win = ep.PeerWindows(comm, cfg.M, cfg.hidden, T * cfg.k * world,
                             barrier="host" if gloo else "device", device=device)

        def p2p_step(i, x=None, lg=None, a=None):
            if x is None:
                x, lg, a = inputs[i % n_inputs]
            return shards[i % len(shards)].forward_p2p(win, x, lg, ladder, i % NUM_LAYERS, NUM_LAYERS,
                                                       phase, attn_mass=a)

        p2p_step(0)   # one step, then check every rank's status before timing anything
        torch.cuda.synchronize()
        st = torch.tensor([float(win.status.item())], device=device if not gloo else "cpu",
                          dtype=torch.float64)
        torch.distributed.all_reduce(st, op=torch.distributed.ReduceOp.MAX)
        if st.item() != 0:
            raise RuntimeError("peer-memory step reported status %d" % int(st.item()))
        for i in range(1, args.warmup):
            p2p_step(i)
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.distributed.barrier()
        torch.cuda.synchronize()
        with ClockSampler(torch.cuda.current_device()) as clk_p2p:
            q0.record()
            for i in range(K):
                p2p_step(args.warmup + i)
            q1.record()
            torch.cuda.synchronize()
        torch.distributed.barrier()
        qms = _max_over_ranks(q0.elapsed_time(q1), device)
        st = torch.tensor([float(win.status.item())], device=device if not gloo else "cpu",
                          dtype=torch.float64)
        torch.distributed.all_reduce(st, op=torch.distributed.ReduceOp.MAX)
        p2p = {"value": T * K * world / (qms / 1e3), "unit": "tokens/s", "ms_per_step": qms / K,
               "scaling": "weak", "barrier": win.barrier_mode, "status": int(st.item()),
               "note": "dymoe_ep_dispatch / dymoe_ep_combine over peer windows (CUDA IPC), "
                       "no NCCL on the data path; 3 flag barriers + 1 count read per step"}
    except Exception as ex:   # reported, never fatal for the NCCL line
        p2p = {"error": "%s: %s" % (type(ex).__name__, str(ex)[:300])}
    use_p2p = p2p is not None and "error" not in p2p and p2p["status"] == 0 and \
        args.ep_main != "nccl" and (torch.distributed.get_backend() == "nccl" or args.ep_main == "p2p")
    nccl_line = {"value": value, "unit": "tokens/s", "ms_per_step": nccl_ms / K, "scaling": "weak",
                 "note": "NCCL all_to_all_single dispatch / combine (counts exchanged first)"}
    if use_p2p:
        ms, value, clk = qms, p2p["value"], clk_p2p

    # ---------------- end-to-end: per step the rank's inputs come from pinned host memory and
    # its output goes back to the host, inside the timed region
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
        j = (args.warmup + i) % n_inputs
        dx.copy_(hx[j], non_blocking=True)
        dl.copy_(hl[j], non_blocking=True)
        if phase == d.DYMOE_PREFILL:
            da.copy_(ha[j], non_blocking=True)
        if use_p2p:
            y, _ = p2p_step(args.warmup + i, dx, dl, da)
        else:
            y, _ = shards[(args.warmup + i) % len(shards)].forward(
                dx, dl, ladder, (args.warmup + i) % NUM_LAYERS, NUM_LAYERS, phase, attn_mass=da)
        hy.copy_(y, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e2e = {"value": T * K * world / (_max_over_ranks(e0.elapsed_time(e1), device) / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    if win is not None:
        torch.distributed.barrier()
        win.close()

    # ---------------- decode, batch replicated on every rank (SURVEY §8e latency variant):
    # the same B tokens everywhere, local experts, one all-reduce of y; strong scaling of one batch
    rep = None
    if phase == d.DYMOE_DECODE:
        xr, lgr, _ = inputs[0]
        _broadcast(xr)
        _broadcast(lgr)
        for i in range(args.warmup):
            shards[i % len(shards)].forward_replicated(xr, lgr, ladder, i % NUM_LAYERS, NUM_LAYERS)
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.distributed.barrier()
        torch.cuda.synchronize()
        r0.record()
        for i in range(K):
            shards[(args.warmup + i) % len(shards)].forward_replicated(
                xr, lgr, ladder, (args.warmup + i) % NUM_LAYERS, NUM_LAYERS)
        r1.record()
        torch.cuda.synchronize()
        torch.distributed.barrier()
        rms = _max_over_ranks(r0.elapsed_time(r1), device)
        rep = {"value": T * K / (rms / 1e3), "unit": "tokens/s", "ms_per_step": rms / K,
               "scaling": "strong", "global_batch": T,
               "note": "the same %d-token batch on every rank; local experts + all-reduce(sum) of y" % T}

    # local FFN roofline (bytes of the local experts actually streamed / FFN time)
    ffn_ms, ffn_bytes, ffn_flops = 0.0, 0.0, 0.0
    for e0, e1, bits, off in ffn_events:
        ffn_ms += e0.elapsed_time(e1)
        b = bits.cpu().numpy()
        o = off.cpu().numpy()
        for e in range(len(o) - 1):
            n = int(o[e + 1] - o[e])
            if n:
                chunks = (n + 7) // 8 if phase == d.DYMOE_DECODE else max(1, (n + 255) // 256)
                ffn_bytes += 3 * cfg.hidden * cfg.ffn * bytes_per_weight(int(b[e])) * chunks
                ffn_flops += 6.0 * cfg.hidden * cfg.ffn * n
    res = None
    if phase == d.DYMOE_DECODE:
        ach = ffn_bytes / max(ffn_ms / 1e3, 1e-12) / 1e9
        roof = {"bound": "hbm", "kernel": "local fused-dequant FFN (k_decode_gemv W13 + W2), rank 0",
                "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s", "frac": ach / peaks["hbm"],
                "traffic": None, "peak_src": peaks["src"]}
    else:
        ach = ffn_flops / max(ffn_ms / 1e3, 1e-12) / 1e12
        pk = peaks["bf16_sus"] or peaks["bf16"]
        roof = {"bound": "tensor", "kernel": "local tcgen05 fused-dequant grouped GEMM, rank 0",
                "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "traffic": None,
                "peak_src": peaks["src"] + " bf16 sustained"}
    if rank == 0:
        res = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K,
               "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "bf16 x int8/int4/int2 (fp32 accum)",
               "data": "synthetic (seeded random-init Mixtral-8x7B-shaped experts, Zipf-skewed router logits)",
               "config": {"workload": wname, "hidden": cfg.hidden, "ffn": cfg.ffn,
                          "experts": cfg.M, "top_k": cfg.k, "tokens_per_step_per_rank": T,
                          "global_batch": T * world,
                          "ladder": {"bits": LADDER_BITS, "lambdas": LADDER_LAMBDAS},
                          "schedule": "layer l = step mod 32 of a 32-layer depth schedule",
                          "weight_copies": args.copies, "l2": "inputs larger than L2 (rotating weight copies)",
                          "parallelism": ("ep%d (experts sharded, peer-memory dispatch/combine kernels)" % world)
                          if use_p2p else ("ep%d (experts sharded, NCCL all-to-all dispatch/combine)" % world)},
               "roofline": roof, "clocks": clk.summary(), "e2e": e2e,
               # libdymoe launches per step and rank: route, score, assign, permute, ep_plan,
               # gather_rows, local permute, active list, W13, W2, reduce / prefill gather,
               # unit-weight reorder, weighted combine (NCCL collectives not counted)
               "gpu_launches": (15 if use_p2p else 13) * K,
               "ep_path": "p2p" if use_p2p else "nccl_all_to_all",
               "ep_replicated_decode": rep, "ep_p2p": p2p, "ep_nccl_all_to_all": nccl_line}
    return res


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
    (profiles/traffic.json, written from profiles/r01_ncu_*.md), with the algorithmic work of
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
        out["attention_mass"] = {"us": us, "TFLOP/s": fl / (us * 1e-6) / 1e12, "H": H, "d": 128,
                                 "note": "two causal Q.K^T passes (row stats, column sums), mma.sync"}
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
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prefill-kernel", default="ss", choices=["ss", "ts"],
                    help="prefill expert GEMM: ss = dequantized weights through shared memory "
                         "(default), ts = the experimental operand-swapped kernel (weights in TMEM)")
    ap.add_argument("--no-graph", action="store_true", help="time the steps call by call instead "
                    "of replaying their CUDA graph (single-GPU decode / prefill / stack workloads)")
    ap.add_argument("--ep-main", default="auto", choices=["auto", "nccl", "p2p"],
                    help="N > 1: the main line's dispatch/combine path (auto: the peer-memory path "
                         "when it runs clean under NCCL, else the NCCL all-to-all)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test hook for several ranks sharing one GPU (collectives staged "
                         "through host memory); never used for reported numbers")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
            raise SystemExit("--workload stack runs on one GPU (the EP stack needs 8 GPUs)")
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
