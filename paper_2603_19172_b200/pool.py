"""HBM-resident mixed-precision expert store driven by the expert pool (PAPER.md
"Mixed-Precision Cache Management").

The paper keeps a VRAM cache of experts at two precisions and streams misses over PCIe.
On B200 every bf16 master can sit in HBM, and the packed formats are what a byte budget has to
hold: at C5 scale (32 Mixtral-shaped layers) all three packed widths of every expert would take
~105 GB on top of the 90 GB of masters.  The store keeps packed formats in one device arena of
`capacity` bytes, managed by the dymoe_pool policy (No Duplication, Precision Promotion,
Conservative Reuse, LRU, pins), and fills misses by runtime quantization (dymoe_quantize) of the
bf16 master straight into the arena slot -- the pool decides when dymoe_quantize runs.

One step of layer l (`forward`):
  1. route / score / assign on the device (libdymoe), the bits read back to the host;
  2. `prepare`: for every routed expert with bits b in {2, 4, 8}: pool lookup; a hit is served by
     the cached format (b' >= b, Conservative Reuse); a miss or promotion inserts (evicting LRU
     entries, whose layer bindings are dropped), quantizes the master into the slot and rebinds
     the expert (dymoe_layer_set_expert).  BF16 requests are served by the masters (outside the
     budget).  Every expert of the step is pinned while the step is prepared;
  3. dymoe_moe_forward with the SERVED widths as forced bits.
`prefetch(l, bits, stream, after)` runs step 2 ahead of time on a SIDE stream (
PAPER.md "Phase-Adaptive Prefetcher"): the look-ahead predictor dymoe_predict_next
(Eqs. 6-8) names layer l+1's likely critical experts from layer l's hidden state, and their
high-precision formats are quantized into the arena while layer l's FFN runs on the main stream
(`PrefetchingStack` below).  Ordering: the side stream first waits for `after` (an event the main
stream recorded once every kernel of earlier layers was queued before it), so an eviction never
overwrites a slot an in-flight kernel still reads; the experts of the running layer are pinned
while the prefetch decides its evictions; layer l+1's step waits for the prefetch's completion
event before it touches the pool.

Host-offload variant (the paper's own setting): with masters in (pinned)
host memory, BF16 becomes a pool format like the packed ones (the arena holds a bf16 copy), and a
miss first copies the expert's bf16 master host -> device into a staging buffer (the paper's
PCIe / C2C transfer), then quantizes it into the slot (or, for BF16, copies it into the slot).
All device work is ordered on one stream, so an arena range is only overwritten after the kernels
already queued on it have read it.
"""
import contextlib

import torch

from . import dymoe as d

_ALIGN = 256


def _al(n):
    return (n + _ALIGN - 1) // _ALIGN * _ALIGN


class ExpertStore:
    def __init__(self, masters, k_route, hidden, ffn, capacity, device="cuda"):
        """masters: [layer][expert] dicts with bf16 'w1', 'w3' [F, Hd] and 'w2' [Hd, F], on the
        device (packed formats pooled) or in host memory (host-offload: every format pooled,
        pinned host tensors recommended).  capacity: arena bytes."""
        self.masters = masters
        self.k, self.hidden, self.ffn = k_route, hidden, ffn
        self.L, self.M = len(masters), len(masters[0])
        self.device = torch.device(device)
        self.host = not masters[0][0]["w1"].is_cuda
        self.arena = torch.empty(capacity, dtype=torch.uint8, device=device)
        self.pool = d.Pool(capacity)
        if self.host:
            # staging buffers for an expert's three bf16 matrices, one set per stream that loads
            # (the main stream's demand misses and the prefetch side stream run concurrently);
            # reuse within a stream is stream-ordered
            self.stages = {}
            self.layers = [d.MoELayer([{} for _ in ml], k_route, hidden, ffn) for ml in masters]
        else:
            self.layers = [d.MoELayer([dict(e) for e in ml], k_route, hidden, ffn) for ml in masters]
        self.bound = [[None] * self.M for _ in range(self.L)]   # (bits, offset) of the bound format
        self.stats = dict(hits=0, misses=0, promotions=0, evictions=0, quantized_bytes=0,
                          prefetched=0, prefetch_hits=0)
        self.ready = {}            # layer -> event: its prefetch has finished on the side stream
        self.prefetched = set()    # (layer, expert) inserted by a prefetch, not yet used by a step

    # ------------------------------------------------------------------ arena layout
    def _shapes(self):
        return (("w1", self.ffn, self.hidden), ("w3", self.ffn, self.hidden), ("w2", self.hidden, self.ffn))

    def entry_bytes(self, bits):
        n = 0
        for _, N, K in self._shapes():
            if bits == 16:
                n += _al(N * K * 2)
            else:
                n += _al(N * K * bits // 8) + _al(N * (K // d.GROUP) * 4) + _al(N * (K // d.GROUP))
        return n

    def _views(self, off, bits):
        if bits == 16:
            out = {}
            for name, N, K in self._shapes():
                out[name] = self.arena[off:off + N * K * 2].view(torch.bfloat16).view(N, K)
                off += _al(N * K * 2)
            return out
        q = {}
        for name, N, K in self._shapes():
            nc, ns, nz = N * K * bits // 8, N * (K // d.GROUP) * 4, N * (K // d.GROUP)
            codes = self.arena[off:off + nc].view(torch.int32).view(N, K * bits // 32)
            off += _al(nc)
            scales = self.arena[off:off + ns].view(torch.float32).view(N, K // d.GROUP)
            off += _al(ns)
            zeros = self.arena[off:off + nz].view(N, K // d.GROUP)
            off += _al(nz)
            q[name] = (codes, scales, zeros)
        return q

    def _bind(self, l, e, bits, off, stream):
        ex = {} if self.host else dict(self.masters[l][e])
        if bits == 16:
            ex.update(self._views(off, 16))
        elif bits is not None:
            ex["q%d" % bits] = self._views(off, bits)
        self.layers[l].set_expert(e, ex, stream=stream)
        self.bound[l][e] = (bits, off) if bits is not None else None

    # ------------------------------------------------------------------ policy
    def prepare(self, l, bits, stream=None, keep_pinned=(), prefetch=False):
        """Make every requested width of layer l resident; returns the served widths (list).
        keep_pinned: (layer, expert) keys held pinned while this call decides evictions."""
        served = [0] * self.M
        pinned = []
        for key in keep_pinned:
            self.pool.pin(*key)
            pinned.append(key)
        try:
            for e, b in enumerate(bits):
                b = int(b)
                if b == 0 or (b == 16 and not self.host):
                    served[e] = b
                    continue
                out, sb, off = self.pool.lookup(l, e, b)
                if out == d.POOL_HIT:
                    if not prefetch:
                        self.stats["hits"] += 1
                        if (l, e) in self.prefetched:
                            self.stats["prefetch_hits"] += 1
                            self.prefetched.discard((l, e))
                    if self.bound[l][e] != (sb, off):
                        self._bind(l, e, sb, off, stream)
                else:
                    if prefetch:
                        self.stats["prefetched"] += 1
                        self.prefetched.add((l, e))
                    else:
                        self.stats["misses" if out == d.POOL_MISS else "promotions"] += 1
                    off, evicted = self.pool.insert(l, e, b, self.entry_bytes(b))
                    for (l2, e2) in evicted:
                        self.stats["evictions"] += 1
                        self.prefetched.discard((l2, e2))
                        self._bind(l2, e2, None, None, stream)
                    views = self._views(off, b)
                    src = self._source(l, e, stream)
                    if b == 16:
                        with (torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()):
                            for n in ("w1", "w3", "w2"):
                                views[n].copy_(src[n], non_blocking=True)
                    else:
                        jobs = [(src[n], b, views[n]) for n in ("w1", "w3", "w2")]
                        d.dymoe_quantize_batched(jobs, stream=stream)
                        self.stats["quantized_bytes"] += self.entry_bytes(b)
                    self._bind(l, e, b, off, stream)
                    sb = b
                self.pool.pin(l, e)
                pinned.append((l, e))
                served[e] = sb
        finally:
            for (pl, pe) in pinned:
                self.pool.unpin(pl, pe)
        return served

    def prefetch(self, l, bits, stream, after=None, keep_pinned=()):
        """prepare(l, bits) on the side `stream` (after the main stream's event `after`); the
        completion event is what layer l's step waits for (`ready[l]`)."""
        if after is not None:
            stream.wait_event(after)
        self.prepare(l, bits, stream, keep_pinned=keep_pinned, prefetch=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        self.ready[l] = ev
        return ev

    def wait_ready(self, l, stream=None):
        ev = self.ready.pop(l, None)
        if ev is not None:
            (stream or torch.cuda.current_stream()).wait_event(ev)

    def _source(self, l, e, stream):
        """The expert's bf16 master on the device (host-offload: copied into the staging buffer)."""
        if not self.host:
            return self.masters[l][e]
        st = stream or torch.cuda.current_stream()
        key = st.cuda_stream
        if key not in self.stages:
            # allocated on the stream that uses it: the caching allocator may hand a block freed
            # on stream S to a new allocation made on S while S's queued kernels still read it
            # (safe only for work ordered on S) -- a side-stream staging buffer carved from a
            # main-stream block would be overwritten by H2D copies that race those kernels
            with torch.cuda.stream(st):
                self.stages[key] = {n: torch.empty(N, K, dtype=torch.bfloat16, device=self.device)
                                    for n, N, K in self._shapes()}
        stage = self.stages[key]
        with (torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()):
            for n in ("w1", "w3", "w2"):
                stage[n].copy_(self.masters[l][e][n], non_blocking=True)
        self.stats["h2d_bytes"] = self.stats.get("h2d_bytes", 0) + sum(t.numel() * 2 for t in stage.values())
        return stage

    def assigned_bits(self, l, x, logits, ladder, num_layers, phase, attn_mass=None, k_tokens=0):
        """Steps route -> score -> assign of dymoe_moe_forward (libdymoe kernels); returns the
        bits on the host (the one synchronisation of a pooled step)."""
        idx, _, _ = d.dymoe_route(logits, self.k)
        imp, _ = d.dymoe_score(phase, self.M, self.k, topk_idx=idx, attn_mass=attn_mass,
                               logits=logits, k_tokens=k_tokens)
        bits = d.dymoe_assign_bits(imp, l, num_layers, ladder, self.k)[0]
        active = torch.zeros(self.M, dtype=torch.bool, device=bits.device)
        active[idx.reshape(-1).long()] = True
        return (bits * active.to(bits.dtype)).cpu().tolist(), bits

    def forward(self, l, x, logits, ladder, num_layers, phase=d.DYMOE_DECODE, attn_mass=None,
                k_tokens=0, stream=None, out=None, out_dtype=d.DYMOE_OUT_F32, residual=None):
        """One pooled layer step; returns (y, served widths, requested widths, forced widths the
        forward ran with: served for routed experts, assigned for the others)."""
        want, bits_dev = self.assigned_bits(l, x, logits, ladder, num_layers, phase, attn_mass, k_tokens)
        # a prefetch of this layer must have finished writing before this stream touches the
        # arena (its own loads may evict and overwrite, its FFN reads); the routing above did not
        self.wait_ready(l, stream)
        served = self.prepare(l, want, stream)
        # experts not routed this step keep their assigned width (they run no rows)
        forced = [s if w else int(b) for s, w, b in zip(served, want, bits_dev.cpu().tolist())]
        forced_t = torch.tensor(forced, dtype=torch.uint8, device=x.device)
        y, _ = self.layers[l].forward(x, logits, ladder, l, num_layers, phase=phase,
                                      attn_mass=attn_mass, k_tokens=k_tokens, forced_bits=forced_t,
                                      stream=stream, out=out, out_dtype=out_dtype, residual=residual)
        return y, served, want, forced


class PrefetchingStack:
    """A layer stack (stack.MoEStack's block: RMSNorm -> router -> MoE -> residual) over an
    ExpertStore whose arena is smaller than the packed formats of the whole stack, with the
    paper's look-ahead prefetcher (Eqs. 6-8, steps 5-6 of
    P:203): at layer l, dymoe_predict_next on l's normed hidden state with layer l+1's gate ranks
    the experts of l+1 (prefill: token frequency, Eq. 7; decode: the predicted gate, Eq. 8); the
    predicted experts' formats at the widths layer l+1's schedule gives their ranks (Eq. 5 tier
    counts: the top t_1 -- the paper's critical experts -- at the top tier) are quantized into
    the arena on a side stream while layer l's FFN runs on the main stream.  prefetch=False: every format is
    loaded on demand (the baseline the overlap is measured against).  policy "critical": only the
    top t_1 predicted experts, at the top tier (the paper's prefetch of the critical experts);
    "tiered": every predicted expert at its predicted tier."""

    def __init__(self, store, gates, policy="critical"):
        assert policy in ("critical", "tiered")
        self.store = store
        self.gates = gates
        self.policy = policy
        self.L, self.M, self.k = store.L, store.M, store.k
        self.side = torch.cuda.Stream(device=store.device)

    def forward(self, x, ladder, phase=d.DYMOE_DECODE, attn_masses=None, prefetch=True, eps=1e-5,
                trace=False):
        s = self.store
        main = torch.cuda.current_stream()
        T = x.shape[0]
        u = torch.empty_like(x)
        bufs = (torch.empty_like(x), torch.empty_like(x))
        logits = torch.empty(T, self.M, dtype=torch.float32, device=x.device)
        cur, out_trace = x, [] if trace else None
        for l in range(self.L):
            start = torch.cuda.Event()
            start.record(main)                   # every kernel of layers < l is queued before it
            wg, beta = self.gates[l]
            d.dymoe_rmsnorm(cur, eps, out=u)
            d.dymoe_gate_logits(u, wg, beta, out=logits)
            nxt = bufs[l & 1]
            a = attn_masses[l] if attn_masses is not None else None
            req = None
            if prefetch and l + 1 < self.L:
                # Eqs. 6-8 on the device; the requests are read back before this layer's FFN is
                # queued (the step synchronises for its own bits anyway), so nothing waits for it.
                # Every predicted expert is requested at the width layer l+1's schedule gives its
                # predicted rank (Eq. 5 tier counts at depth l+1): the critical ones at the top
                # tier as in the paper, the rest at theirs -- prefetching everything
                # at the top width would overfill the byte budget and evict the next layers
                tiers = d.dymoe_tier_counts(l + 1, self.L, ladder, self.M, self.k)
                # decode: at most T k experts can be active (B = 1: the top-k of Eq. 8)
                t = self.M if phase == d.DYMOE_PREFILL else min(self.M, T * self.k)
                if self.policy == "critical":
                    t = max(1, min(t, tiers[0] if tiers else self.M))
                ex, _, _ = d.dymoe_predict_next(phase, u, self.gates[l + 1][0], self.k, t)
                req = [0] * self.M
                for rank, e in enumerate(ex.cpu().tolist()):
                    tier = sum(1 for t in tiers if rank >= t)
                    req[e] = ladder.bits[tier]
            y, served, want, forced = s.forward(l, u, logits, ladder, self.L, phase=phase,
                                                attn_mass=a, out=nxt, out_dtype=d.DYMOE_OUT_BF16,
                                                residual=cur)
            if req is not None:
                keep = [(l, e) for e in range(self.M) if want[e]]
                s.prefetch(l + 1, req, self.side, after=start, keep_pinned=keep)
            if trace:
                out_trace.append((cur.clone(), u.clone(), logits.clone(), list(forced), list(served)))
            cur = nxt
        return cur, out_trace
