"""Group-wise quantization, packing and dequantization, SURVEY §8c O4/O5.

Test infrastructure only (see oracle/__init__.py).

Paper: experts are quantized with GPTQ at 4 and 2 bits (AWQ/HQQ
"seamlessly").  Reading D14: the runtime quantizer is
round-to-nearest on GPTQ's asymmetric min-max grid (min/max widened to include 0,
integer zero point, an all-zero group uses (-1, +1)); GPTQ's Hessian error
feedback needs calibration data and is out of scope.  Reading D15: groups of
G = 128 consecutive weights along K (the input dimension) of each row; scale fp32,
zero uint8.  Reading D16: the reciprocal form q = rint(w * (1/s)) + z.

All arithmetic below is IEEE float32, one rounding per operation, exactly in the
order written (NumPy float32 array ops do not contract into FMAs):
  w32  = float32(bf16 w)
  mn   = min(0, min w32);  mx = max(0, max w32)
  s    = (mx - mn) / maxq                       maxq = 2**b - 1
         if s < 2**-126 (incl. mn = mx = 0):  mn, mx = -1, +1 and s recomputed (D14b)
  inv  = 1 / s
  z    = rint(-mn * inv)                        (half to even) -> uint8
  q    = clip(rint(w32 * inv) + z, 0, maxq)
Pack: code k of a row goes to word k // (32/b), bits (k % (32/b)) * b, LSB first.
Dequant (O5 / R17): deq = RNE_bf16( (q - z) * RNE_bf16(s) ).
"""

import numpy as np

from .bf16 import round_bf16

QBITS = (2, 4, 8)


def _check(bits, K, group):
    if bits not in QBITS:
        raise ValueError("bits: quantized widths are 2, 4 or 8")
    if group <= 0 or K % group != 0:
        raise ValueError("group: K must be a multiple of the group size")


def quantize_groups(w, bits, group=128):
    """w: float32 [N, K] holding bf16 values.  Returns (q uint8 [N,K], s f32 [N,K/G], z u8 [N,K/G])."""
    w = np.asarray(w, dtype=np.float32)
    N, K = w.shape
    _check(bits, K, group)
    maxq = np.float32(2 ** bits - 1)
    g = w.reshape(N, K // group, group)
    zero32 = np.float32(0.0)
    mn = np.minimum(zero32, g.min(axis=2))
    mx = np.maximum(zero32, g.max(axis=2))
    s = ((mx - mn).astype(np.float32) / maxq).astype(np.float32)
    # D14b: a group whose scale is zero or below the smallest normal float32 (2**-126;
    # 1/s could overflow) uses the all-zero rule (-1, +1).  This covers mn == mx == 0.
    degen = s < np.float32(2.0 ** -126)
    mn = np.where(degen, np.float32(-1.0), mn).astype(np.float32)
    mx = np.where(degen, np.float32(1.0), mx).astype(np.float32)
    s = ((mx - mn).astype(np.float32) / maxq).astype(np.float32)
    inv = (np.float32(1.0) / s).astype(np.float32)
    z = np.rint(((-mn).astype(np.float32) * inv).astype(np.float32)).astype(np.float32)
    prod = (g * inv[:, :, None]).astype(np.float32)
    q = np.rint(prod).astype(np.float32) + z[:, :, None]
    q = np.clip(q, 0, maxq).astype(np.uint8).reshape(N, K)
    return q, s.astype(np.float32), z.astype(np.uint8)


def pack(q, bits):
    """q uint8 [N, K] -> uint32 [N, K*bits/32], LSB-first."""
    q = np.asarray(q, dtype=np.uint64)
    N, K = q.shape
    per = 32 // bits
    if K % per:
        raise ValueError("K: must be a multiple of 32/bits")
    q = q.reshape(N, K // per, per)
    words = np.zeros((N, K // per), dtype=np.uint64)
    for i in range(per):
        words |= q[:, :, i] << np.uint64(i * bits)
    return words.astype(np.uint32)


def unpack(codes, bits, K):
    """uint32 [N, K*bits/32] -> uint8 [N, K]."""
    codes = np.asarray(codes, dtype=np.uint64)
    N = codes.shape[0]
    per = 32 // bits
    mask = np.uint64((1 << bits) - 1)
    out = np.zeros((N, codes.shape[1], per), dtype=np.uint8)
    for i in range(per):
        out[:, :, i] = ((codes >> np.uint64(i * bits)) & mask).astype(np.uint8)
    return out.reshape(N, codes.shape[1] * per)[:, :K]


def quantize(w, bits, group=128):
    """Quantize + pack one matrix: returns (codes u32, scales f32, zeros u8)."""
    q, s, z = quantize_groups(w, bits, group)
    return pack(q, bits), s, z


def dequant(codes, scales, zeros, bits, K, group=128):
    """O5: RNE_bf16((q - z) * RNE_bf16(s)) as float64 [N, K]."""
    q = unpack(codes, bits, K).astype(np.float64)
    N = q.shape[0]
    s_b = round_bf16(np.asarray(scales, dtype=np.float32).astype(np.float64))
    z = np.asarray(zeros, dtype=np.float64)
    qz = q.reshape(N, K // group, group) - z[:, :, None]
    return round_bf16(qz * s_b[:, :, None]).reshape(N, K)


def bytes_per_weight(bits, group=128):
    """Algorithmic storage per weight: b/8 + (4 + 1)/G for quantized, 2 for bf16, 0 for skip."""
    if bits == 16:
        return 2.0
    if bits == 0:
        return 0.0
    return bits / 8.0 + 5.0 / group
