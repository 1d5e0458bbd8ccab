"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NO arithmetic of the method (no routing, scoring, scheduling,
quantization or FFN); it only draws random tensors with the shapes and value
distributions of the paper's workloads (recipe: DESIGN.md §5).
The gate GEMM that turns hidden states into router logits is outside the path
(reading R19) and is part of input generation.

Everything is drawn with a seeded ``torch.Generator`` on the requested device (CPU
for the small parity configs, CUDA for the full-size bench so that 1.4 G weights do
not cross PCIe); the same (seed, device) always yields the same tensors.
"""

from dataclasses import dataclass, replace
import math

import torch


@dataclass(frozen=True)
class MoEConfig:
    name: str
    M: int          # experts per layer
    k: int          # routing top-k
    hidden: int     # Hd
    ffn: int        # F
    T: int          # tokens per step (B for decode)
    heads: int = 32  # H, attention heads feeding Eq. 1
    group: int = 128
    layers: int = 32

    def with_tokens(self, T):
        return replace(self, T=T)


# BASELINE.json configs[0..4]
CONFIGS = {
    "tiny": MoEConfig("tiny", M=8, k=2, hidden=256, ffn=512, T=16),
    # a small fine-grained-style layer (many experts, top-4) for multi-rank parity tests
    "ep_small": MoEConfig("ep_small", M=16, k=4, hidden=256, ffn=384, T=40),
    "mixtral_decode": MoEConfig("mixtral_decode", M=8, k=2, hidden=4096, ffn=14336, T=8),
    "mixtral_prefill": MoEConfig("mixtral_prefill", M=8, k=2, hidden=4096, ffn=14336, T=2048),
    "finegrained": MoEConfig("finegrained", M=64, k=6, hidden=2048, ffn=1408, T=2048),
    "stack": MoEConfig("stack", M=8, k=2, hidden=4096, ffn=14336, T=8, layers=32),
}

ZIPF_ALPHA = 1.2       # SPEC default skew
HH_FRAC = 0.2          # heavy-hitter token fraction


def generator(seed, device="cpu"):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def expert_weights(cfg, seed, device="cpu", experts=None):
    """bf16 masters per expert: W1, W3 ~ N(0, 1/Hd) [F, Hd]; W2 ~ N(0, 1/F) [Hd, F]."""
    g = generator(seed * 1000 + 7, device)
    out = []
    ids = range(cfg.M) if experts is None else experts
    last = cfg.M if experts is None else max(experts) + 1   # same stream, stop early
    for e in range(last):
        sd_in, sd_out = 1.0 / math.sqrt(cfg.hidden), 1.0 / math.sqrt(cfg.ffn)
        w1 = torch.randn(cfg.ffn, cfg.hidden, generator=g, device=device).mul_(sd_in)
        w3 = torch.randn(cfg.ffn, cfg.hidden, generator=g, device=device).mul_(sd_in)
        w2 = torch.randn(cfg.hidden, cfg.ffn, generator=g, device=device).mul_(sd_out)
        if e in ids:
            out.append(dict(w1=w1.to(torch.bfloat16), w3=w3.to(torch.bfloat16),
                            w2=w2.to(torch.bfloat16)))
        del w1, w3, w2
    return out


def hidden_states(cfg, seed, device="cpu", T=None):
    """x ~ N(0, 1) rounded to bf16 (post-RMSNorm scale), [T, Hd]."""
    g = generator(seed * 1000 + 11, device)
    T = cfg.T if T is None else T
    return torch.randn(T, cfg.hidden, generator=g, device=device).to(torch.bfloat16)


def router_logits(cfg, x, seed, device="cpu"):
    """l = x W_g^T + beta, W_g ~ N(0, 1/Hd); beta_{pi(r)} = -alpha ln(r+1) (Zipf, seed-permuted)."""
    g = generator(seed * 1000 + 13, device)
    wg = torch.randn(cfg.M, cfg.hidden, generator=g, device=device) / math.sqrt(cfg.hidden)
    perm = torch.randperm(cfg.M, generator=g, device=device)
    beta = torch.empty(cfg.M, device=device)
    beta[perm] = -ZIPF_ALPHA * torch.log(torch.arange(cfg.M, device=device, dtype=torch.float32) + 1.0)
    return (x.float() @ wg.t() + beta).contiguous()


def stack_gate(cfg, layer, seed, device="cpu"):
    """Router of stack layer `layer`: (W_g bf16 [M, Hd] ~ N(0, 1/Hd), beta f32 [M]) with
    beta_{pi(r)} = -alpha ln(r+1) (Zipf, permutation drawn per layer so the hot experts move
    with depth)."""
    g = generator(seed * 1000 + 29 + 7919 * layer, device)
    wg = (torch.randn(cfg.M, cfg.hidden, generator=g, device=device) / math.sqrt(cfg.hidden))
    perm = torch.randperm(cfg.M, generator=g, device=device)
    beta = torch.empty(cfg.M, device=device)
    beta[perm] = -ZIPF_ALPHA * torch.log(torch.arange(cfg.M, device=device, dtype=torch.float32) + 1.0)
    return wg.to(torch.bfloat16).contiguous(), beta.contiguous()


def attention_mass(cfg, seed, device="cpu", T=None):
    """a[h][i] >= 0, fp32 [H, T]: 20% heavy tokens ~ U(4,8)(1+0.1 N(0,1)), rest U(0,1)."""
    g = generator(seed * 1000 + 17, device)
    T = cfg.T if T is None else T
    H = cfg.heads
    heavy = torch.rand(T, generator=g, device=device) < HH_FRAC
    base = torch.rand(H, T, generator=g, device=device)
    hv = (4.0 + 4.0 * torch.rand(H, T, generator=g, device=device)) * \
         (1.0 + 0.1 * torch.randn(H, T, generator=g, device=device))
    a = torch.where(heavy[None, :], hv.clamp_min(0.0), base)
    return a.contiguous()


def layer_inputs(cfg, seed, device="cpu", T=None):
    """(x bf16 [T,Hd], logits f32 [T,M], attn_mass f32 [H,T]) for one step."""
    x = hidden_states(cfg, seed, device, T)
    return x, router_logits(cfg, x, seed, device), attention_mass(cfg, seed, device, x.shape[0])


def random_logits(T, M, seed, device="cpu", ties=False):
    """Plain N(0,1) logits; with ties=True values are drawn from a 4-point set so that
    equal logits (and -0.0 vs +0.0) occur often."""
    g = generator(seed * 1000 + 19, device)
    if ties:
        pts = torch.tensor([-0.0, 0.0, 1.0, -1.0], device=device)
        return pts[torch.randint(0, 4, (T, M), generator=g, device=device)].contiguous()
    return torch.randn(T, M, generator=g, device=device).contiguous()


def random_matrix_bf16(N, K, seed, device="cpu", kind="normal"):
    """Weight-like bf16 matrices for quantizer tests, including edge-case groups."""
    g = generator(seed * 1000 + 23, device)
    if kind == "normal":
        w = torch.randn(N, K, generator=g, device=device)
    elif kind == "positive":
        w = torch.rand(N, K, generator=g, device=device) + 0.01
    elif kind == "negative":
        w = -(torch.rand(N, K, generator=g, device=device) + 0.01)
    elif kind == "zeros":
        w = torch.zeros(N, K, device=device)
    elif kind == "tiny":
        w = torch.randn(N, K, generator=g, device=device) * 1e-38   # bf16 subnormals
    elif kind == "mixed":
        w = torch.randn(N, K, generator=g, device=device)
        w[:, : K // 4] = 0.0
        w[::3, K // 4: K // 2] = -0.0
        w[1::2, K // 2: 3 * K // 4] *= 1e-3
    else:
        raise ValueError(kind)
    return w.to(torch.bfloat16).contiguous()
