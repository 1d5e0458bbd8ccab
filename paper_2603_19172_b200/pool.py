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
`prefetch(l, bits)` runs step 2 ahead of time (e.g. for the widths dymoe_predict_next predicts
for the next layer), on the caller's stream.

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
            # one staging buffer for an expert's three bf16 matrices (reused, stream-ordered)
            self.stage = {n: torch.empty(N, K, dtype=torch.bfloat16, device=device)
                          for n, N, K in self._shapes()}
            self.layers = [d.MoELayer([{} for _ in ml], k_route, hidden, ffn) for ml in masters]
        else:
            self.layers = [d.MoELayer([dict(e) for e in ml], k_route, hidden, ffn) for ml in masters]
        self.bound = [[None] * self.M for _ in range(self.L)]   # (bits, offset) of the bound format
        self.stats = dict(hits=0, misses=0, promotions=0, evictions=0, quantized_bytes=0)

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
    def prepare(self, l, bits, stream=None):
        """Make every requested width of layer l resident; returns the served widths (list)."""
        served = [0] * self.M
        pinned = []
        try:
            for e, b in enumerate(bits):
                b = int(b)
                if b == 0 or (b == 16 and not self.host):
                    served[e] = b
                    continue
                out, sb, off = self.pool.lookup(l, e, b)
                if out == d.POOL_HIT:
                    self.stats["hits"] += 1
                    if self.bound[l][e] != (sb, off):
                        self._bind(l, e, sb, off, stream)
                else:
                    self.stats["misses" if out == d.POOL_MISS else "promotions"] += 1
                    off, evicted = self.pool.insert(l, e, b, self.entry_bytes(b))
                    for (l2, e2) in evicted:
                        self.stats["evictions"] += 1
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

    prefetch = prepare

    def _source(self, l, e, stream):
        """The expert's bf16 master on the device (host-offload: copied into the staging buffer)."""
        if not self.host:
            return self.masters[l][e]
        with (torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()):
            for n in ("w1", "w3", "w2"):
                self.stage[n].copy_(self.masters[l][e][n], non_blocking=True)
        self.stats["h2d_bytes"] = self.stats.get("h2d_bytes", 0) + sum(t.numel() * 2 for t in self.stage.values())
        return self.stage

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
                k_tokens=0, stream=None):
        """One pooled layer step; returns (y, served widths, requested widths, forced widths the
        forward ran with: served for routed experts, assigned for the others)."""
        want, bits_dev = self.assigned_bits(l, x, logits, ladder, num_layers, phase, attn_mass, k_tokens)
        served = self.prepare(l, want, stream)
        # experts not routed this step keep their assigned width (they run no rows)
        forced = [s if w else int(b) for s, w, b in zip(served, want, bits_dev.cpu().tolist())]
        forced_t = torch.tensor(forced, dtype=torch.uint8, device=x.device)
        y, _ = self.layers[l].forward(x, logits, ladder, l, num_layers, phase=phase,
                                      attn_mass=attn_mass, k_tokens=k_tokens, forced_bits=forced_t,
                                      stream=stream)
        return y, served, want, forced
