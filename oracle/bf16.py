"""Round-to-nearest-even onto the bfloat16 grid, evaluated on float64 values.

Test infrastructure only (see oracle/__init__.py).

bfloat16 = 1 sign bit, 8 exponent bits (bias 127), 7 stored mantissa bits, i.e. 8
significant bits for normal numbers and a fixed spacing of 2**-133 below the
smallest normal 2**-126.  Rounding is to nearest, ties to even (IEEE 754 default).
This is the rounding point the contract places on dequantized weights
 and on the SwiGLU intermediate h (O6).

Implemented directly from that definition with frexp/ldexp in float64 -- no double
rounding through float32.  Pinned in tests/test_oracle_bf16.py against hand-worked
ties and against torch's float32->bfloat16 cast on float32 inputs.
"""

import numpy as np

_MANT_BITS = 8          # significant bits of a normal bfloat16
_EMIN = -126            # exponent of the smallest normal (value 2**-126)
_SUB_STEP_EXP = _EMIN - (_MANT_BITS - 1)   # subnormal spacing 2**-133
_MAX = float.fromhex("0x1.fep127")          # largest finite bfloat16


def round_bf16(v):
    """Return float64 array of the bfloat16 values nearest to ``v`` (ties to even)."""
    v = np.asarray(v, dtype=np.float64)
    out = np.zeros_like(v)
    nz = v != 0.0
    m, e = np.frexp(v[nz])              # v = m * 2**e, 0.5 <= |m| < 1
    # normal range: |v| >= 2**-126  <=>  e - 1 >= -126
    normal = (e - 1) >= _EMIN
    r = np.empty_like(m)
    # keep 8 significant bits: m * 2**8 in [128, 256), round half to even
    r[normal] = np.ldexp(np.rint(np.ldexp(m[normal], _MANT_BITS)), e[normal] - _MANT_BITS)
    vs = v[nz][~normal]
    r[~normal] = np.ldexp(np.rint(np.ldexp(vs, -_SUB_STEP_EXP)), _SUB_STEP_EXP)
    if np.any(np.abs(r) > _MAX):
        # values that round above the largest finite bf16 overflow to inf
        r = np.where(np.abs(r) > _MAX, np.sign(r) * np.inf, r)
    out[nz] = r
    return out


def is_bf16(v):
    """True where ``v`` is exactly representable in bfloat16."""
    v = np.asarray(v, dtype=np.float64)
    return round_bf16(v) == v
