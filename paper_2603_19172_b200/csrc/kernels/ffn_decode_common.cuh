// Register-level building blocks of the decode fused-dequant GEMV (ffn_decode.cu): traits per
// width, 128-bit loads, LOP3/PRMT dequant into mma.sync A fragments, matching B fragments, the
// swizzled x layout, and the cost-proportional allocation of virtual CTAs to experts.
#pragma once
#include "../dymoe_internal.cuh"

namespace dymoe {
namespace dec {

template <int BITS>
struct WT {
  static constexpr int CODES = 128 / BITS;   // k values per lane per row per chunk
  static constexpr int CHUNK_K = 4 * CODES;  // k per chunk (a lane quad covers 64 bytes)
  static constexpr int STEPS = CODES / 4;    // mma k16 steps per chunk
  static constexpr int XU4 = CODES / 8;      // uint4 of x per lane per chunk
  static constexpr int GPQ = BITS == 2 ? 2 : 1;   // quantization groups a lane quad spans per chunk
};

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxTok = 8;      // tokens per pass (mma N)

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_f32(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t lop_or_and(uint32_t x, uint32_t mask, uint32_t orv) {
  uint32_t r;  // (x & mask) | orv in one LOP3
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
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t word(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

struct DQ {
  uint32_t ss, zz;    // bf16x2 (s, s) and (128+z, 128+z)
  uint32_t zz1, zz2;  // Int2: (32+z, 32+z) and (8+z, 8+z)
  float sf, zf;       // Int8: bf16(s) as float, 2^23 + z
};

// A-fragment pair (logical k slots lo = {2c, 2c+1}, hi = {2c+8, 2c+9}) for step s of a chunk.
//
// Int4: codes j (bits 4j..4j+3 of each 16-bit half) are shifted down and OR-ed into the mantissa
// of bf16 128 (exponent 7, ulp 1): 128 + q exactly.  (A code at bits 4..7 would reach the
// exponent's lowest bit, so every code but the lowest needs its shift.)
// Int2: no shift for codes at bits 2k..2k+1 (k = 0, 1, 2) of a half: OR-ed into the mantissa of
// bf16 2^(7-2k) (ulp 4^-k) they read as 2^(7-2k) + q exactly, and subtracting bf16(2^(7-2k) + z)
// gives q - z exactly; codes 3-5 / 6-7 of a half come from one shift by 6 / 12.  So a word of 16
// Int2 codes needs 2 shifts instead of 7.
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
    const int j = 2 * (s & 3);   // codes j (lo) and j + 1 (hi) of each half
    const uint32_t y0 = x, y1 = x >> 6, y2 = x >> 12;
    uint32_t v[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int jj = j + t;
      const int k = jj < 3 ? jj : jj < 6 ? jj - 3 : jj - 6;
      const uint32_t y = jj < 3 ? y0 : jj < 6 ? y1 : y2;
      const uint32_t mask = 0x00030003u << (2 * k);
      const uint32_t magic = 0x43004300u - (uint32_t)k * 0x01000100u;
      const uint32_t zz = k == 0 ? dq.zz : k == 1 ? dq.zz1 : dq.zz2;
      v[t] = bf2_mul(bf2_sub(lop_or_and(y, mask, magic), zz), dq.ss);
    }
    lo = v[0];
    hi = v[1];
  } else {  // 8
    // q - z exact in fp32 (2^23 + q minus 2^23 + z), taken to bf16x2 exactly (|q - z| <= 255
    // has 8 significant bits), then one HMUL2 per pair gives RNE((q - z)·s) (D17)
    const uint32_t x = word(w, s);
#ifndef DYMOE_I8_PRMT_PACK
    // the two subtractions as one packed FADD2 and the exact bf16x2 pack as one F2FP, so that a
    // pair costs 2 ALU instructions (the magic PRMTs) instead of 3: the Int8 loop is bound by the
    // ALU pipe (ncu: PRMT at the top of the stall samples)
    float2 z2 = make_float2(-dq.zf, -dq.zf);
    float d0, d1, d2, d3;
    {
      uint64_t r, a, zz;
      asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(prmt(x, 0x4B000000u, 0x7440u)), "r"(prmt(x, 0x4B000000u, 0x7441u)));
      asm("mov.b64 %0, {%1, %2};" : "=l"(zz) : "f"(z2.x), "f"(z2.y));
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(zz));
      asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(r));
      asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(prmt(x, 0x4B000000u, 0x7442u)), "r"(prmt(x, 0x4B000000u, 0x7443u)));
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(zz));
      asm("mov.b64 {%0, %1}, %2;" : "=f"(d2), "=f"(d3) : "l"(r));
    }
    lo = bf2_mul(pack_bf2(d0, d1), dq.ss);   // q - z has <= 8 significant bits: the pack is exact
    hi = bf2_mul(pack_bf2(d2, d3), dq.ss);
#else
    const float d0 = __fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7440u)), dq.zf);
    const float d1 = __fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7441u)), dq.zf);
    const float d2 = __fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7442u)), dq.zf);
    const float d3 = __fsub_rn(__uint_as_float(prmt(x, 0x4B000000u, 0x7443u)), dq.zf);
    // q - z is a small integer (<= 8 significant bits): its fp32 low half is zero, so the bf16
    // pair is just the two high halves (one PRMT instead of an F2FP conversion)
    lo = bf2_mul(prmt(__float_as_uint(d0), __float_as_uint(d1), 0x7632u), dq.ss);
    hi = bf2_mul(prmt(__float_as_uint(d2), __float_as_uint(d3), 0x7632u), dq.ss);
#endif
  }
}

// x granules per block and mma steps per block: a block of GPB granules (8 k values each) of the
// lane's x feeds SPB consecutive k16 steps.
template <int BITS>
struct XB {
  static constexpr int GPB = BITS == 2 ? 2 : 1;
  static constexpr int SPB = BITS == 2 ? 4 : 2;
  static constexpr int NB = WT<BITS>::STEPS / SPB;
};

// B fragment (x in a_frag's k order) for step ss of a block, from the block's x granules.  The x
// staging already permuted the elements of each granule into that order (x_perm), so a fragment is
// two words of a granule at every width.
template <int BITS>
__device__ __forceinline__ void b_frag(const uint4 (&xb)[XB<BITS>::GPB], int ss, uint32_t& b0,
                                       uint32_t& b1) {
  if constexpr (BITS == 2) {
    b0 = word(xb[ss >> 1], 2 * (ss & 1));
    b1 = word(xb[ss >> 1], 2 * (ss & 1) + 1);
  } else {
    b0 = word(xb[0], 2 * ss);
    b1 = word(xb[0], 2 * ss + 1);
  }
}

// Element order of the staged x granules: a_frag's step s pairs, per lane, k values that are not
// adjacent in x (Int4: codes j and j + 4 of a byte pair; Int2: the same code position of two
// consecutive granules), so the staging stores
//   Int4: granule (e0 .. e7) as (e0 e4 e1 e5 e2 e6 e3 e7);
//   Int2: granule pair A, C as (a0 c0 a1 c1 a2 c2 a3 c3), (a4 c4 a5 c5 a6 c6 a7 c7) (half 0, 1);
//   BF16 / Int8: unchanged.
template <int BITS>
__device__ __forceinline__ uint4 x_perm(const uint4& a, const uint4& c, int half) {
  if constexpr (BITS == 4) {
    return make_uint4(prmt(a.x, a.z, 0x5410u), prmt(a.x, a.z, 0x7632u), prmt(a.y, a.w, 0x5410u),
                      prmt(a.y, a.w, 0x7632u));
  } else if constexpr (BITS == 2) {
    const uint32_t a0 = half ? a.z : a.x, a1 = half ? a.w : a.y;
    const uint32_t c0 = half ? c.z : c.x, c1 = half ? c.w : c.y;
    return make_uint4(prmt(a0, c0, 0x5410u), prmt(a0, c0, 0x7632u), prmt(a1, c1, 0x5410u),
                      prmt(a1, c1, 0x7632u));
  } else {
    return a;
  }
}

struct Alloc {   // compact: it shares the 227 KB shared-memory budget with the rings
  int n_act;
  int units_total;                               // <= max(grid, M) < 2^16
  uint8_t expert[DYMOE_MAX_EXPERTS];             // M <= 256
  uint8_t bits[DYMOE_MAX_EXPERTS];               // the expert's width, by list position
  uint16_t first_unit[DYMOE_MAX_EXPERTS + 1];
};
// scratch of compute_alloc (lives in shared memory the pipeline has not started using yet)
struct AllocScratch {
  long long cost[DYMOE_MAX_EXPERTS];
  int list[DYMOE_MAX_EXPERTS];
  int rows[DYMOE_MAX_EXPERTS];
  int bits[DYMOE_MAX_EXPERTS];
};

// Relative time to stream one expert matrix set at width b (per 8-token chunk), measured on B200
// with every expert forced to one width (tools/decode_width_sweep.py): the narrow widths are
// bound by dequant issue slots rather than bytes, so they cost more than their bytes suggest.
__device__ __forceinline__ int wcost(int b, bool w13) {
  if (w13) return b == 16 ? 259 : b == 8 ? 162 : b == 4 ? 115 : 103;
  return b == 16 ? 256 : b == 8 ? 179 : b == 4 ? 130 : 129;
}

// Cost-proportional allocation of `units_total` units to the active experts, every active
// expert >= 1 unit: with C_i the exclusive prefix of the costs in list order and R = U - n,
// first_unit[i] = i + floor(R * C_i / total) (so expert i gets 1 + floor(R C_{i+1} / total) -
// floor(R C_i / total) units and the total is exactly U).  Warp 0, all 32 lanes.  The active
// list, every expert's row count and every width are loaded in ONE round of independent loads
// (lanes stride over the M experts; the list length is loaded alongside) into shared scratch,
// then each lane takes a contiguous block of the list and the prefix is a warp scan over the
// blocks -- the kernel's whole ramp is this allocation plus the x staging, so dependent global
// round trips here cost every CTA directly (tools/dec_trace.py: 2.0 us with three dependent
// rounds).  Every CTA computes the identical allocation; it only partitions tiles, never the
// arithmetic.
__device__ void compute_alloc(const FfnArgs& a, int units_grid, bool w13, Alloc& A,
                              AllocScratch& X) {
  const int lane = threadIdx.x & 31;
  const int M = a.M;
  const int n = __ldg(a.active_list);
#pragma unroll 8
  for (int i = lane; i < M; i += 32) {
    const int l = __ldg(a.active_list + 1 + i);
    const int o0 = __ldg(a.expert_off + i), o1 = __ldg(a.expert_off + i + 1);
    const int b = __ldg(a.bits + i);
    X.list[i] = l;
    X.rows[i] = o1 - o0;
    X.bits[i] = b;
  }
  __syncwarp();
  const int per = (n + 31) / 32;
  const int i0 = lane * per, i1 = min(n, i0 + per);
  long long local = 0;
  for (int i = i0; i < i1; ++i) {
    const int e = X.list[i];
    const long long c = (long long)wcost(X.bits[e], w13) * ((X.rows[e] + kMaxTok - 1) / kMaxTok);
    A.expert[i] = (uint8_t)e;
    A.bits[i] = (uint8_t)X.bits[e];
    X.cost[i] = c;
    local += c;
  }
  long long incl = local;   // inclusive warp scan of the block sums
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const long long total = __shfl_sync(0xffffffffu, incl, 31);
  const int U = units_grid > n ? units_grid : n;
  const long long R = U - n;
  long long cum = incl - local;
  for (int i = i0; i < i1; ++i) {
    A.first_unit[i] = (uint16_t)(i + (total > 0 ? (int)(R * cum / total) : 0));
    cum += X.cost[i];
  }
  if (lane == 0) {
    A.n_act = n;
    A.units_total = U;
    A.first_unit[n] = (uint16_t)U;
  }
}


}  // namespace dec
}  // namespace dymoe
