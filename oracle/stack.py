"""A stack of MoE layers on the residual stream (BASELINE.json configs[4]:
"full 32-layer Mixtral-8x7B-shaped stack, random weights, depth-adaptive bits").

Test infrastructure only (see oracle/__init__.py).

Per layer l = 0 .. L-1 (attention omitted; a synthetic attention mass per layer),
a Mixtral block's MoE half on the bf16 residual stream (pre-norm, unit RMSNorm weight):
  u_l      = RNE_bf16(x_l / sqrt(mean(x_l^2) + eps))     RMSNorm (fp64, one rounding);
  logits_l = u_l W_g^(l)T + beta^(l)   the router on the layer's own hidden state: the
                                       Eq. 6 gate product evaluated exactly (prefetch.gate_logits,
                                       reading P1) plus the bias, in fp64;
  y_l      = moe.moe_forward(u_l, logits_l, experts_l, l, L, ...)   (fp64, the whole layer with
                                       the depth-aware bits of Eq. 4-5 at depth l);
  x_{l+1}  = RNE_bf16(x_l + y_l)       (the residual stream is bf16; x_l + y_l in fp64, one
                                       rounding).
Without the norm the stream of a random-init stack explodes (SwiGLU is quadratic in its input).
Pinned in tests/test_oracle_stack.py: RMSNorm closed forms (constant rows, power-of-two scale
invariance, unit mean square); zero expert outputs leave the stream unchanged; the bias add; an
all-BF16 k = M stack equals an independent torch fp64 chain of RMSNorm + dense softmax-weighted
SwiGLU mixtures (the textbook reduction of moe.moe_forward, layer by layer).
"""

import numpy as np

from . import bf16 as _bf16
from . import moe as _moe
from . import prefetch as _prefetch


def router_logits(x, w_gate, bias=None):
    """float64 [T, M]: the exact router logits x W_g^T + bias (prefetch.gate_logits + bias, fp64;
    the bias add of two such values is within 2^-53 relative of exact)."""
    lg = _prefetch.gate_logits(x, w_gate)
    if bias is not None:
        lg = lg + np.asarray(bias, dtype=np.float64)[None, :]
    return lg


EPS = 1e-5


def rmsnorm(x, eps=EPS):
    """u = RNE_bf16(x / sqrt(mean(x^2) + eps)) per row, fp64: float64 array of bf16 values."""
    x = np.asarray(x, dtype=np.float64)
    return _bf16.round_bf16(x / np.sqrt((x * x).mean(axis=1, keepdims=True) + eps))


def residual(x, y):
    """x_{l+1} = RNE_bf16(x_l + y_l): float64 array of bf16 values."""
    return _bf16.round_bf16(np.asarray(x, dtype=np.float64) + np.asarray(y, dtype=np.float64))


def stack_layer(x, w_gate, bias, experts, l, L, ladder, k_route, phase="decode", attn_mass=None,
                k_tokens=None, u=None, forced_bits=None):
    """One layer of the stack: returns (x_next float64 [T, Hd] of bf16 values, logits, the
    moe_forward result dict with 'u' added).  u: the normed input to use instead of rmsnorm(x)
    (teacher forcing in parity tests: the GPU's u, checked separately against rmsnorm(x)).
    forced_bits: widths to use instead of the schedule's (moe.moe_forward's option)."""
    u = rmsnorm(x) if u is None else np.asarray(u, dtype=np.float64)
    lg = router_logits(u, w_gate, bias)
    out = _moe.moe_forward(u.astype(np.float32), lg, experts, l, L, ladder, k_route, phase=phase,
                           attn_mass=attn_mass, k_tokens=k_tokens, forced_bits=forced_bits)
    out["u"] = u
    return residual(x, out["y"]), lg, out


def stack_forward(x, gates, experts_per_layer, ladder, k_route, phase="decode", attn_masses=None):
    """The whole stack: gates = [(w_gate, bias)] per layer.  Returns the final x and the list of
    per-layer (x_in, logits, bits)."""
    L = len(gates)
    trace = []
    for l in range(L):
        a = attn_masses[l] if attn_masses is not None else None
        x_next, lg, out = stack_layer(x, gates[l][0], gates[l][1], experts_per_layer[l], l, L,
                                      ladder, k_route, phase, a)
        trace.append((np.asarray(x, np.float64), lg, out["bits"]))
        x = x_next
    return x, trace
