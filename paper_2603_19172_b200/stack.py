"""MoEStack: L DyMoE layers on the bf16 residual stream (BASELINE.json
configs[4]: a 32-layer Mixtral-8x7B-shaped stack with depth-adaptive bits).

Per layer l (attention omitted, as in C5; a Mixtral block's pre-norm MoE half):
  u_l      = RMSNorm(x_l)                   dymoe_rmsnorm (unit weight, bf16 out)
  logits_l = u_l W_g^(l)T + beta^(l)       dymoe_gate_logits (P:111 router on the layer's own
                                            hidden state; fp32 under the reading-P1 error bound, one fp32 bias add)
  x_{l+1}  = bf16(x_l + MoE_l(u_l))         dymoe_moe_forward at depth (l, L) -- route, score,
                                            assign (Eq. 4-5 at depth l), permute, fused-dequant
                                            FFN, combine -- with the residual added in the
                                            combine (dymoe_fwd_opts.residual) and a bf16 output.
Everything runs in libdymoe kernels on the caller's stream (argument marshalling only here); one
workspace serves every layer (same shapes), two bf16 stream buffers alternate, one holds u.
"""
import torch

from . import dymoe as d


class MoEStack:
    def __init__(self, layers, gates, k_route, hidden, ffn):
        """layers: per layer the expert list MoELayer takes (packed widths; bf16 masters only
        if the ladder uses the BF16 tier); gates: per layer (W_g bf16 [M, Hd], beta f32 [M])."""
        assert len(layers) == len(gates) and len(layers) >= 1
        self.layers = [d.MoELayer(ex, k_route, hidden, ffn) for ex in layers]
        self.gates = gates
        self.L = len(layers)
        self.M = self.layers[0].M
        self.k = k_route
        self.hidden = hidden
        self.ffn = ffn

    def workspace(self, T, device="cuda"):
        return self.layers[0].workspace(T, device)

    def forward(self, x, ladder, phase=d.DYMOE_DECODE, attn_masses=None, ws=None, bufs=None,
                logits=None, trace=False, stream=None, first_layer=0, n_layers=None, eps=1e-5):
        """x bf16 [T, Hd] (not modified).  Returns (x_L bf16 [T, Hd], per-layer trace or None):
        with trace=True, [(x_l, u_l, logits_l, bits_l, topk_idx_l)] copies for parity tests.  bufs: three
        bf16 [T, Hd] buffers (stream ping-pong, normed input)."""
        T = x.shape[0]
        dev = x.device
        ws = ws if ws is not None else self.workspace(T, dev)
        if bufs is None:
            bufs = (torch.empty_like(x), torch.empty_like(x), torch.empty_like(x))
        u = bufs[2]
        if logits is None:
            logits = torch.empty(T, self.M, dtype=torch.float32, device=dev)
        out_trace = [] if trace else None
        cur = x
        n = self.L - first_layer if n_layers is None else n_layers
        for i in range(n):
            l = first_layer + i
            wg, beta = self.gates[l]
            d.dymoe_rmsnorm(cur, eps, out=u, stream=stream)
            d.dymoe_gate_logits(u, wg, beta, out=logits, stream=stream)
            nxt = bufs[i & 1]
            self.layers[l].forward(u, logits, ladder, l, self.L, phase=phase,
                                   attn_mass=attn_masses[l] if attn_masses is not None else None,
                                   out_dtype=d.DYMOE_OUT_BF16, ws=ws, out=nxt, residual=cur,
                                   stream=stream)
            if trace:
                v = self.layers[l].views(T, ws)
                out_trace.append((cur.clone(), u.clone(), logits.clone(), v["bits"].clone(),
                                  v["topk_idx"].clone()))
            cur = nxt
        return cur, out_trace


class EPStack:
    """The C5 stack with every MoE layer expert-parallel (BASELINE.json configs[4]: "full
    32-layer Mixtral-8x7B-shaped stack ... expert-parallel on 8xB200"): each rank holds, per
    layer, the block of experts it owns (ep.owned_range) and its own tokens' residual stream; per
    layer RMSNorm and the router run on the rank's tokens, then dymoe_moe_forward_ep (global
    importance, exchange, owners' FFN, combine with the residual, bf16 stream out).  ONE
    dymoe_ep handle (one window / communicator) serves all layers: the local expert table of the
    layer is passed per call.  Marshalling only, like MoEStack."""

    def __init__(self, ep_layer, local_layers, gates):
        """ep_layer: an ep.EPLayer (its handle and transport set-up; its own local table is the
        first layer's); local_layers: per layer the expert list of this rank's owned experts;
        gates: per layer (W_g bf16 [M, Hd], beta f32 [M])."""
        self.ep = ep_layer
        self.layers = [d.MoELayer(ex, 1, ep_layer.hidden, ep_layer.ffn) for ex in local_layers]
        self.gates = gates
        self.L = len(local_layers)
        self.M, self.k, self.hidden = ep_layer.M, ep_layer.k, ep_layer.hidden

    def forward(self, x, ladder, phase=d.DYMOE_DECODE, transport=d.DYMOE_EP_PEER,
                attn_masses=None, ws=None, bufs=None, logits=None, trace=False, stream=None,
                eps=1e-5, T_peer_max=0):
        T = x.shape[0]
        ws = ws if ws is not None else self.ep.workspace(T, T_peer_max, device=x.device)
        if bufs is None:
            bufs = (torch.empty_like(x), torch.empty_like(x), torch.empty_like(x))
        u = bufs[2]
        if logits is None:
            logits = torch.empty(T, self.M, dtype=torch.float32, device=x.device)
        out_trace = [] if trace else None
        cur = x
        for l in range(self.L):
            wg, beta = self.gates[l]
            d.dymoe_rmsnorm(cur, eps, out=u, stream=stream)
            d.dymoe_gate_logits(u, wg, beta, out=logits, stream=stream)
            nxt = bufs[l & 1]
            self.ep.forward(u, logits, ladder, l, self.L, phase, transport=transport,
                            attn_mass=attn_masses[l] if attn_masses is not None else None,
                            T_peer_max=T_peer_max, out_dtype=d.DYMOE_OUT_BF16, residual=cur,
                            ws=ws, out=nxt, stream=stream, local=self.layers[l])
            if trace:
                v = self.ep.views(T, ws, T_peer_max)
                out_trace.append((cur.clone(), u.clone(), logits.clone(), v["bits"].clone(),
                                  v["topk_idx"].clone()))
            cur = nxt
        return cur, out_trace
