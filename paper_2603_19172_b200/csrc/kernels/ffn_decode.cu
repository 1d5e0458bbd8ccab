// Decode expert FFN (row a7): fused-dequant SwiGLU GEMV for <= 8 rows per expert, sm_100a.
//
// Paper: P:203 step 4 (executor on a unified mixed-precision weight set), P:312 (Int4/Int2
// experts, skip), P:356 (decode is dominated by fetching expert weights).  Readings D13, D17,
// D18, O6: A = x·deq(W1)^T, B = x·deq(W3)^T in fp32, h = RNE_bf16(silu(A)·B),
// y = h·deq(W2)^T in fp32, deq = RNE_bf16((q - z)·RNE_bf16(s)).
//
// Roofline: HBM.  Every active expert's packed W1/W3/W2 is streamed exactly once per step
// (3·Hd·F·(b/8 + 5/128) bytes).  At Int2 there are only ~2 ALU issue slots per weight at the
// HBM rate, so:
//  * the multiply-adds run on the tensor cores: mma.sync m16n8k16 with 16 weight rows as A and
//    the (up to 8) tokens as the N=8 columns of B, fp32 accumulation;
//  * dequant is done in registers straight into A fragments: Int2/Int4 codes are OR-ed into the
//    mantissa of bf16 128.0 (one LOP3 per 2 weights gives 128+q exactly), then HSUB2 (128+z)
//    gives q-z exactly and HMUL2 by bf16(s) gives RNE((q-z)·s) — bit-identical to D17;
//    Int8 uses the fp32 magic 2^23+q, FADD, FMUL (exact) and one cvt.rn.bf16x2;
//  * the dot product is permutation-invariant in k, so each lane's A fragment takes the codes in
//    the order the LOP3 extracts them (code i and i+4 of a word, i.e. no shuffling of weights),
//    and the matching x values are permuted instead (PRMT on the x registers, which are reused
//    across all row tiles of the warp).
// Layout per chunk: a lane quad (4 lanes) reads 64 contiguous bytes of one weight row (one
// uint4 per lane); 8 quads cover rows g = 0..7 and a second uint4 covers rows g + 8.  A CTA owns
// 16·RT output rows of one expert; its NW warps split K round-robin by chunk and reduce the
// partial 16x8 tiles through shared memory in warp order (deterministic).  W13: both W1 and W3
// tiles for the same rows, SwiGLU applied in the reduction epilogue, h written as bf16.
// Grid: (rows / (16·RT), number of active experts) — CTAs of a quantized width stream 4-8x
// fewer bytes than BF16 ones; the hardware block scheduler balances them.
#include "../dymoe_internal.cuh"

namespace dymoe {
namespace {

template <int BITS>
struct WT {
  static constexpr int CODES = 128 / BITS;   // k values per lane per row per chunk
  static constexpr int CHUNK_K = 4 * CODES;  // k per chunk (a lane quad)
  static constexpr int STEPS = CODES / 4;    // mma k16 steps per chunk
  static constexpr int XU4 = CODES / 8;      // uint4 of x per lane per chunk
};

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint32_t lop_or_and(uint32_t x, uint32_t mask, uint32_t orv) {
  uint32_t r;  // (x & mask) | orv  -> a single LOP3
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(x), "r"(mask), "r"(orv));
  return r;
}

__device__ __forceinline__ uint32_t bf2_sub(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&a),
                             *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t bf2_mul(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmul2(*reinterpret_cast<__nv_bfloat162*>(&a),
                             *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 r = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t word(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Per-row dequant parameters (packed bf16x2 for Int2/Int4; fp32 pair for Int8).
struct DQ {
  uint32_t ss, zz;  // bf16x2 (s,s), (128+z, 128+z)
  float sf, zf;     // Int8: s as float (bf16-rounded), 2^23 + z
};

template <int BITS>
__device__ __forceinline__ DQ make_dq(float s, uint32_t z) {
  DQ d;
  const __nv_bfloat16 sb = __float2bfloat16_rn(s);
  const uint16_t sbits = *reinterpret_cast<const uint16_t*>(&sb);
  d.ss = (uint32_t)sbits | ((uint32_t)sbits << 16);
  const uint32_t zb = 0x4300u | z;  // bf16(128 + z), exact for z < 128
  d.zz = zb | (zb << 16);
  d.sf = __bfloat162float(sb);
  d.zf = __uint_as_float(0x4B000000u | z);
  return d;
}

// A-fragment pair (logical slots lo = {2c, 2c+1}, hi = {2c+8, 2c+9}) for step s of a chunk.
template <int BITS>
__device__ __forceinline__ void a_frag(const uint4& w, const DQ& dq, int s, uint32_t& lo,
                                       uint32_t& hi) {
  if constexpr (BITS == 16) {
    lo = word(w, 2 * s);
    hi = word(w, 2 * s + 1);
  } else if constexpr (BITS == 4) {
    const uint32_t x = word(w, s >> 1);
    const int sh = 8 * (s & 1);
    lo = bf2_mul(bf2_sub(lop_or_and(x >> sh, 0x000F000Fu, 0x43004300u), dq.zz), dq.ss);
    hi = bf2_mul(bf2_sub(lop_or_and(x >> (sh + 4), 0x000F000Fu, 0x43004300u), dq.zz), dq.ss);
  } else if constexpr (BITS == 2) {
    const uint32_t x = word(w, s >> 2);
    const int sh = 4 * (s & 3);
    lo = bf2_mul(bf2_sub(lop_or_and(x >> sh, 0x00030003u, 0x43004300u), dq.zz), dq.ss);
    hi = bf2_mul(bf2_sub(lop_or_and(x >> (sh + 2), 0x00030003u, 0x43004300u), dq.zz), dq.ss);
  } else {  // 8
    const uint32_t x = word(w, s);
    const float q0 = __fmul_rn(__fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7440u)), dq.zf), dq.sf);
    const float q1 = __fmul_rn(__fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7441u)), dq.zf), dq.sf);
    const float q2 = __fmul_rn(__fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7442u)), dq.zf), dq.sf);
    const float q3 = __fmul_rn(__fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7443u)), dq.zf), dq.sf);
    lo = pack_bf2(q0, q1);
    hi = pack_bf2(q2, q3);
  }
}

// B fragment (x values permuted to match a_frag's k order) for step s.
template <int BITS>
__device__ __forceinline__ void b_frag(const uint4 (&xv)[WT<BITS>::XU4], int s, uint32_t& b0,
                                       uint32_t& b1) {
  if constexpr (BITS == 16) {
    b0 = word(xv[0], 2 * s);
    b1 = word(xv[0], 2 * s + 1);
  } else if constexpr (BITS == 8) {
    b0 = word(xv[s >> 1], 2 * (s & 1));
    b1 = word(xv[s >> 1], 2 * (s & 1) + 1);
  } else if constexpr (BITS == 4) {
    const uint4& u = xv[s >> 1];
    const int j = s & 1;
    const uint32_t a = word(u, j), c = word(u, j + 2);
    b0 = prmt(a, c, 0x5410u);
    b1 = prmt(a, c, 0x7632u);
  } else {  // 2
    const int q = s >> 2, j = s & 3;
    const uint32_t a = word(xv[2 * q], j), c = word(xv[2 * q + 1], j);
    b0 = prmt(a, c, 0x5410u);
    b1 = prmt(a, c, 0x7632u);
  }
}

constexpr int kNW = 8;  // warps per CTA (split-K)

template <bool W13>
struct Cfg {
  static constexpr int RT = 2;               // 16-row tiles per CTA
  static constexpr int NM = W13 ? 2 : 1;     // matrices (W1+W3 or W2)
  static constexpr int ROWS = 16 * RT;
};

template <bool W13, int BITS>
__device__ __forceinline__ void gemv_body(const FfnArgs& a, int e, int row0, int tok0, int nt,
                                          float* red) {
  using C = Cfg<W13>;
  using T = WT<BITS>;
  constexpr int RT = C::RT, NM = C::NM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int K = W13 ? a.Hd : a.F;
  const DevExpert& E = a.experts[e];
  const int wi = width_index(BITS);

  const uint8_t* mat_base[NM];
  const float* sc_base[NM];
  const uint8_t* zr_base[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int mi = W13 ? m : 2;
    if constexpr (BITS == 16) {
      mat_base[m] = reinterpret_cast<const uint8_t*>(E.w[mi]);
      sc_base[m] = nullptr;
      zr_base[m] = nullptr;
    } else {
      mat_base[m] = reinterpret_cast<const uint8_t*>(E.q[wi][mi].codes);
      sc_base[m] = E.q[wi][mi].scales;
      zr_base[m] = E.q[wi][mi].zeros;
    }
  }
  const size_t row_bytes = (size_t)K * BITS / 8;
  const int gpr = K / DYMOE_GROUP;

  // x row of this lane's B column (token g)
  const bool tok_ok = g < nt;
  const uint16_t* xrow = nullptr;
  if (tok_ok) {
    const int r = tok0 + g;
    xrow = W13 ? a.x + (size_t)a.perm_token[r] * a.Hd : a.h + (size_t)r * a.F;
  }

  float acc[RT][NM][4];
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[t][m][i] = 0.f;

  const int nchunks = (K + T::CHUNK_K - 1) / T::CHUNK_K;
  for (int ci = warp; ci < nchunks; ci += kNW) {
    const int kb = ci * T::CHUNK_K + c * T::CODES;  // this lane's first k
    const bool k_ok = kb < K;
    uint4 wv[RT][NM][2];
#pragma unroll
    for (int t = 0; t < RT; ++t)
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = row0 + t * 16 + g + 8 * h;
          wv[t][m][h] = k_ok ? ld_stream(mat_base[m] + row * row_bytes + (size_t)kb * BITS / 8)
                             : make_uint4(0, 0, 0, 0);
        }
    DQ dq[RT][NM][2];
    if constexpr (BITS != 16) {
      const int grp = k_ok ? kb / DYMOE_GROUP : 0;
#pragma unroll
      for (int t = 0; t < RT; ++t)
#pragma unroll
        for (int m = 0; m < NM; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = row0 + t * 16 + g + 8 * h;
            const float s = __ldg(sc_base[m] + (size_t)row * gpr + grp);
            const uint32_t z = __ldg(zr_base[m] + (size_t)row * gpr + grp);
            dq[t][m][h] = make_dq<BITS>(s, z);
          }
    }
    uint4 xv[T::XU4];
#pragma unroll
    for (int i = 0; i < T::XU4; ++i)
      xv[i] = (tok_ok && k_ok) ? __ldg(reinterpret_cast<const uint4*>(xrow + kb) + i)
                               : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int s = 0; s < T::STEPS; ++s) {
      uint32_t b0, b1;
      b_frag<BITS>(xv, s, b0, b1);
#pragma unroll
      for (int t = 0; t < RT; ++t)
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          uint32_t glo, ghi, g8lo, g8hi;
          a_frag<BITS>(wv[t][m][0], dq[t][m][0], s, glo, ghi);
          a_frag<BITS>(wv[t][m][1], dq[t][m][1], s, g8lo, g8hi);
          if (!k_ok) glo = ghi = g8lo = g8hi = 0u;
          mma16816(acc[t][m], glo, g8lo, ghi, g8hi, b0, b1);
        }
    }
  }
  // partial tiles -> shared memory: red[warp][t*NM+m][row16][tok8]
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      float* p = red + ((warp * RT + t) * NM + m) * 128;
      p[g * 8 + 2 * c] = acc[t][m][0];
      p[g * 8 + 2 * c + 1] = acc[t][m][1];
      p[(g + 8) * 8 + 2 * c] = acc[t][m][2];
      p[(g + 8) * 8 + 2 * c + 1] = acc[t][m][3];
    }
}

template <bool W13>
__global__ void __launch_bounds__(kNW * 32) k_decode_gemv(const FfnArgs a) {
  using C = Cfg<W13>;
  constexpr int ROWS = C::ROWS, NM = C::NM, RT = C::RT;
  __shared__ float red[kNW * RT * NM * 128];
  const int slot = blockIdx.y;
  if (slot >= a.active_list[0]) return;
  const int e = a.active_list[1 + slot];
  const int be = a.bits[e];
  const int row0 = blockIdx.x * ROWS;
  const int N = W13 ? a.F : a.Hd;
  const int r_lo = a.expert_off[e], r_hi = a.expert_off[e + 1];
  if (be == 0 || r_hi <= r_lo || row0 >= N) return;

  // residency check (device-side fault -> status word, zero outputs)
  const DevExpert& E = a.experts[e];
  bool resident = true;
  for (int m = 0; m < NM; ++m) {
    const int mi = W13 ? m : 2;
    if (be == 16) resident &= E.w[mi] != nullptr;
    else resident &= width_index(be) >= 0 && E.q[width_index(be)][mi].codes != nullptr;
  }
  if (!resident) {
    if (threadIdx.x == 0 && a.status) atomicOr(a.status, (unsigned)DYMOE_STATUS_WIDTH_NOT_RESIDENT);
    for (int r = r_lo; r < r_hi; ++r)
      for (int i = threadIdx.x; i < ROWS; i += blockDim.x) {
        if (W13) a.h[(size_t)r * a.F + row0 + i] = 0;
        else a.y_perm[(size_t)r * a.Hd + row0 + i] = 0.f;
      }
    return;
  }

  for (int tok0 = r_lo; tok0 < r_hi; tok0 += 8) {
    const int nt = min(8, r_hi - tok0);
    switch (be) {
      case 2: gemv_body<W13, 2>(a, e, row0, tok0, nt, red); break;
      case 4: gemv_body<W13, 4>(a, e, row0, tok0, nt, red); break;
      case 8: gemv_body<W13, 8>(a, e, row0, tok0, nt, red); break;
      default: gemv_body<W13, 16>(a, e, row0, tok0, nt, red); break;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < ROWS * 8; o += blockDim.x) {
      const int tok = o / ROWS, rl = o - tok * ROWS;
      if (tok >= nt) continue;
      const int t = rl >> 4, r16 = rl & 15;
      float s0 = 0.f, s1 = 0.f;
      for (int w = 0; w < kNW; ++w) {
        const float* p = red + ((w * RT + t) * NM) * 128 + r16 * 8 + tok;
        s0 = __fadd_rn(s0, p[0]);
        if (NM == 2) s1 = __fadd_rn(s1, p[128]);
      }
      const size_t r = (size_t)(tok0 + tok);
      if (W13) {
        const float silu = __fdiv_rn(s0, __fadd_rn(1.f, expf(-s0)));
        const __nv_bfloat16 hv = __float2bfloat16_rn(__fmul_rn(silu, s1));
        a.h[r * a.F + row0 + rl] = *reinterpret_cast<const uint16_t*>(&hv);
      } else {
        a.y_perm[r * a.Hd + row0 + rl] = s0;
      }
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_ffn_decode(const FfnArgs& a, cudaStream_t s, void* const* ev) {
  const int max_active = a.M < a.T * a.k ? a.M : a.T * a.k;
  record_ev(ev, 0, s);
  if (max_active > 0) {
    dim3 g13(a.F / Cfg<true>::ROWS, max_active);
    k_decode_gemv<true><<<g13, kNW * 32, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  record_ev(ev, 1, s);
  if (max_active > 0) {
    dim3 g2(a.Hd / Cfg<false>::ROWS, max_active);
    k_decode_gemv<false><<<g2, kNW * 32, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  record_ev(ev, 2, s);
  return cudaSuccess;
}

}  // namespace dymoe
