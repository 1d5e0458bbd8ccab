// Decode expert FFN (row a7): fused-dequant SwiGLU GEMV for few tokens per expert, sm_100a.
//
// Paper: P:203 step 4 (executor on a unified mixed-precision weight set), P:312 (Int4/Int2
// experts, skip), P:356 (decode is dominated by fetching expert weights).  Readings D13, D17,
// D18, O6: A = x·deq(W1)^T, B = x·deq(W3)^T in fp32, h = RNE_bf16(silu(A)·B),
// y = h·deq(W2)^T in fp32, deq = RNE_bf16((q - z)·RNE_bf16(s)).
//
// Roofline: HBM.  Every active expert's packed W1/W3/W2 is streamed once per 8-token chunk
// (3·Hd·F·(b/8 + 5/128) bytes per expert).
//
// Arithmetic.  At Int2 there are only ~2 ALU issue slots per weight at the HBM rate:
//  * multiply-adds on the tensor cores: mma.sync m16n8k16, 16 weight rows as A, the (<= 8)
//    tokens as the N = 8 columns of B, fp32 accumulation;
//  * dequant in registers straight into A fragments: Int2/Int4 codes are OR-ed into the mantissa
//    of bf16 128.0 (one LOP3 per 2 weights gives 128+q exactly), HSUB2 (128+z) gives q-z
//    exactly, HMUL2 by bf16(s) gives RNE((q-z)·s) — bit-identical to D17.  Int8 uses the fp32
//    magic 2^23+q, FADD, FMUL (exact) and one cvt.rn.bf16x2;
//  * the dot product is permutation-invariant in k, so A fragments take codes in the order the
//    LOP3 extracts them (code i and i+4 of a word) and the x values are permuted to match (PRMT
//    on registers loaded from shared memory).
//
// Work decomposition (one launch per matrix pair, persistent, cost-balanced):
//  * grid = 1 CTA per SM; each CTA walks "virtual CTAs".  Every CTA computes the same
//    allocation of virtual CTAs to the active experts, proportional to each expert's streamed
//    bytes (width x token chunks), so CTAs of Int8 and Int2 experts finish together.
//  * a virtual CTA = (expert, K-slice, range of 16-row tiles).  Its tokens' x slice is staged
//    once in shared memory (XOR-swizzled, conflict-free LDS.128), then the 8 warps split every
//    tile's K round-robin by chunk, and reduce the 16x8 partial tiles through shared memory in
//    warp order (deterministic, double-buffered, one barrier per tile).
//  * each warp streams its chunks through its own cp.async (LDGSTS, L1-bypassing) shared-memory
//    ring of 6 (W1/W3) or 8 (W2) stages, so 5-7 chunks per warp (~10 KB at Int4 for W1+W3) are
//    in flight while it computes; lanes only read back the bytes their own quad copied.
//  * W1/W3 (gate/up): one K-slice (x = 8 x Hd bf16 in smem), SwiGLU applied in the reduction
//    epilogue, h written as bf16.  W2 (down): K = F is split into SK slices (x slice <= 64 KB),
//    each writes fp32 partials y_part[slice]; the combine kernel sums the slices in order.
#include "../dymoe_internal.cuh"

namespace dymoe {
namespace {

template <int BITS>
struct WT {
  static constexpr int CODES = 128 / BITS;   // k values per lane per row per chunk
  static constexpr int CHUNK_K = 4 * CODES;  // k per chunk (a lane quad covers 64 bytes)
  static constexpr int STEPS = CODES / 4;    // mma k16 steps per chunk
  static constexpr int XU4 = CODES / 8;      // uint4 of x per lane per chunk
  // row padding (in 16-byte granules, mod 8) that makes the 2 token rows of an LDS.128 phase
  // hit disjoint bank groups (see x_granule)
  static constexpr int PAD = BITS == 2 ? 4 : BITS == 4 ? 2 : BITS == 8 ? 1 : 4;
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
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t word(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

struct DQ {
  uint32_t ss, zz;  // bf16x2 (s, s) and (128+z, 128+z)
  float sf, zf;     // Int8: bf16(s) as float, 2^23 + z
};
__device__ __forceinline__ DQ make_dq(float s, uint32_t z) {
  DQ d;
  const __nv_bfloat16 sb = __float2bfloat16_rn(s);
  const uint32_t sbits = *reinterpret_cast<const uint16_t*>(&sb);
  d.ss = sbits | (sbits << 16);
  const uint32_t zb = 0x4300u | z;  // bf16(128 + z), exact for z < 128 (Int2/Int4)
  d.zz = zb | (zb << 16);
  d.sf = __bfloat162float(sb);
  d.zf = __uint_as_float(0x4B000000u | z);
  return d;
}

// A-fragment pair (logical k slots lo = {2c, 2c+1}, hi = {2c+8, 2c+9}) for step s of a chunk.
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

// B fragment (x permuted to a_frag's k order) for step s, from the chunk's x registers.
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

// x slice in shared memory: [8 tokens][row_gran granules of 16 B], granule index XOR-swizzled
// with (g >> 3) & 7 so that the 4 lanes of a quad (k offsets c*XU4 granules apart) hit distinct
// bank groups; row_gran = sliceK/8 + PAD puts the second token row of a phase on the other four.
__device__ __forceinline__ int x_granule(int g) { return g ^ ((g >> 3) & 7); }

struct Alloc {
  int n_act;
  int expert[DYMOE_MAX_EXPERTS];
  int first_unit[DYMOE_MAX_EXPERTS + 1];
  int units_total;
  long long cost[DYMOE_MAX_EXPERTS];   // scratch
  long long rem[DYMOE_MAX_EXPERTS];
  int u[DYMOE_MAX_EXPERTS];
};

__device__ __forceinline__ int wcost(int b) { return b == 16 ? 256 : 16 * b + 5; }

// Cost-proportional allocation of `units_total` units to the active experts (largest remainder,
// ties to the lower list index; every active expert gets >= 1 unit).  Thread 0 only.
__device__ void compute_alloc(const FfnArgs& a, int units_grid, Alloc& A) {
  const int n = a.active_list[0];
  A.n_act = n;
  long long* cost = A.cost;
  long long total = 0;
  for (int i = 0; i < n; ++i) {
    const int e = a.active_list[1 + i];
    A.expert[i] = e;
    const int rows = a.expert_off[e + 1] - a.expert_off[e];
    const int chunks = (rows + kMaxTok - 1) / kMaxTok;
    cost[i] = (long long)wcost(a.bits[e]) * chunks;
    total += cost[i];
  }
  const int U = units_grid > n ? units_grid : n;
  A.units_total = U;
  int* u = A.u;
  long long* rem = A.rem;
  int used = 0;
  for (int i = 0; i < n; ++i) {
    const long long num = (long long)(U - n) * cost[i];   // n units reserved (one each)
    u[i] = 1 + (int)(num / total);
    rem[i] = num % total;
    used += u[i];
  }
  while (used < U) {  // hand out the rest by largest remainder
    int best = 0;
    for (int i = 1; i < n; ++i)
      if (rem[i] > rem[best]) best = i;
    u[best] += 1;
    rem[best] = -1;
    ++used;
  }
  int acc = 0;
  for (int i = 0; i < n; ++i) {
    A.first_unit[i] = acc;
    acc += u[i];
  }
  A.first_unit[n] = acc;
}

// Per-warp cp.async (LDGSTS) ring.  One stage = one chunk of this warp:
//   weights: NM*2 uint4 per lane, laid out [item][lane] (conflict-free LDS.128);
//   scales:  [quad][pair] f32 — a quad needs NM*2 (m, h) x GPQ groups pairs, lane c copies
//            pairs c, c + 4 (no redundant copies across the quad);
//   zeros:   [quad][pair] u32 — the aligned word holding that zero byte (byte index kept in a
//            register and shuffled to the reader).
template <int NM>
struct Ring {
  static constexpr int W_BYTES = NM * 2 * 32 * 16;
  static constexpr int S_BYTES = 8 * 8 * 4;   // [quad][pair v < 8] (NM*2 (m,h) x <= 2 groups)
  static constexpr int STAGE = W_BYTES + 2 * S_BYTES;
};
template <bool W13>
struct Pipe {
  static constexpr int STAGES = W13 ? 6 : 8;
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
  return r;
}

// Issue the copies of pipeline item q (tile t0 + q / cmax, this warp's chunk q % cmax) into the
// stage at shared address `st`.
template <int BITS, int NM>
__device__ __forceinline__ void issue_chunk(uint32_t st, const uint8_t* const (&mat)[NM],
                                            const float* const (&scl)[NM],
                                            const uint8_t* const (&zer)[NM], size_t row_bytes,
                                            int gpr, size_t n_groups, int t0, int cmax, int nck,
                                            int kl, int k0, int warp, int lane, int q,
                                            uint32_t& zsel) {
  using Tr = WT<BITS>;
  const int g = lane >> 2, c = lane & 3;
  const int tile = t0 + q / cmax;
  const int ci = warp + kWarps * (q % cmax);
  const int kb = ci * Tr::CHUNK_K + c * Tr::CODES;   // lane's first k within the slice
  if (!(ci < nck)) return;
  const int kg = k0 + kb;
  if (kb < kl) {
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = tile * 16 + g + 8 * h;
        cp_async16(st + ((m * 2 + h) * 32 + lane) * 16,
                   mat[m] + (size_t)row * row_bytes + (size_t)kg * BITS / 8);
      }
  }
  if constexpr (BITS != 16) {
    // the quad needs V = NM*2*GPQ (scale, zero) pairs: (m, h) x the GPQ groups its lanes span
    // (Int2 lanes 0-1 and 2-3 fall in different groups).  Lane c copies pairs v = c, c + 4, ...
    constexpr int NC = NM * 2, GPQ = Tr::GPQ, V = NC * GPQ;
    const int chunk_k0 = k0 + ci * Tr::CHUNK_K;
    zsel = 0;
#pragma unroll
    for (int v = c, i = 0; v < V; v += 4, ++i) {
      const int cc = v % NC, j = v / NC;
      const int m = cc >> 1, h = cc & 1;
      const int row = tile * 16 + g + 8 * h;
      const int kj = chunk_k0 + j * (Tr::CHUNK_K / GPQ);
      if (kj - k0 >= kl) continue;   // group beyond the slice (Int2 tail)
      const size_t gi = (size_t)row * gpr + kj / DYMOE_GROUP;
      const int slot = (g * V + v) * 4;
      cp_async4(st + Ring<NM>::W_BYTES + slot, scl[m] + gi);
      // zero byte: copy its aligned word when that word lies inside the array
      const size_t wbase = gi & ~(size_t)3;
      uint32_t sel;
      if (wbase + 4 <= n_groups) {
        cp_async4(st + Ring<NM>::W_BYTES + Ring<NM>::S_BYTES + slot, zer[m] + wbase);
        sel = (uint32_t)(gi & 3);
      } else {
        sel = 4u + (uint32_t)__ldg(zer[m] + gi);   // tail of the array: plain byte load
      }
      zsel |= sel << (16 * i);
    }
  }
}

// One virtual CTA: expert e, k-slice ks (global k range [k0, k0 + kl)), tiles [t0, t1),
// tokens [tok0, tok0 + nt).  x slice already in smem.
template <bool W13, int BITS>
__device__ __forceinline__ void run_tiles(const FfnArgs& a, int e, int k0, int kl, int t0, int t1,
                                          int tok0, int nt, int ks, const uint4* xs, int row_gran,
                                          float* red, uint32_t ring_base) {
  using Tr = WT<BITS>;
  constexpr int NM = W13 ? 2 : 1;
  constexpr int S = Pipe<W13>::STAGES;
  constexpr int STAGE = Ring<NM>::STAGE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int K = W13 ? a.Hd : a.F;
  const int N = W13 ? a.F : a.Hd;
  const DevExpert& E = a.experts[e];
  const int wi = width_index(BITS);
  const uint8_t* mat[NM];
  const float* scl[NM];
  const uint8_t* zer[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int mi = W13 ? m : 2;
    if constexpr (BITS == 16) {
      mat[m] = reinterpret_cast<const uint8_t*>(E.w[mi]);
      scl[m] = nullptr;
      zer[m] = nullptr;
    } else {
      mat[m] = reinterpret_cast<const uint8_t*>(E.q[wi][mi].codes);
      scl[m] = E.q[wi][mi].scales;
      zer[m] = E.q[wi][mi].zeros;
    }
  }
  const size_t row_bytes = (size_t)K * BITS / 8;
  const int gpr = K / DYMOE_GROUP;
  const size_t n_groups = (size_t)N * gpr;
  const int nck = (kl + Tr::CHUNK_K - 1) / Tr::CHUNK_K;        // chunks per tile (slice)
  const int cmax = (nck + kWarps - 1) / kWarps;               // per warp (same for all warps)
  const int ntiles = t1 - t0;
  const int n_items = ntiles * cmax;
  const uint32_t ring = ring_base + warp * (S * STAGE);
  uint32_t zsel[S];   // per stage: byte index of the zero in its word, or 4 + the byte itself
#pragma unroll
  for (int i = 0; i < S; ++i) zsel[i] = 0;

  float acc[NM][4];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;

#pragma unroll
  for (int p = 0; p < S - 1; ++p) {
    if (p < n_items)
      issue_chunk<BITS, NM>(ring + p * STAGE, mat, scl, zer, row_bytes, gpr, n_groups, t0, cmax,
                            nck, kl, k0, warp, lane, p, zsel[p]);
    cp_commit();
  }

  int tile_seq = 0;
  for (int q0 = 0; q0 < n_items; q0 += S) {
#pragma unroll
    for (int sidx = 0; sidx < S; ++sidx) {
      const int q = q0 + sidx;
      if (q < n_items) {  // uniform across the CTA: n_items is the same for every warp
        // refill the stage consumed in the previous iteration with item q + S - 1
        {
          const int qn = q + S - 1;
          const int sn = (sidx + S - 1) % S;
          if (qn < n_items)
            issue_chunk<BITS, NM>(ring + sn * STAGE, mat, scl, zer, row_bytes, gpr, n_groups, t0,
                                  cmax, nck, kl, k0, warp, lane, qn, zsel[sn]);
          cp_commit();
        }
        cp_wait<S - 1>();
        __syncwarp();
        const uint32_t st = ring + sidx * STAGE;
        const int ci = warp + kWarps * (q % cmax);
        const int kb = ci * Tr::CHUNK_K + c * Tr::CODES;
        const bool ok = ci < nck && kb < kl;
        if (ci < nck) {
          uint4 xv[Tr::XU4];
          const int gbase = kb / 8;
#pragma unroll
          for (int i = 0; i < Tr::XU4; ++i)
            xv[i] = ok ? xs[g * row_gran + x_granule(gbase + i)] : make_uint4(0, 0, 0, 0);
          DQ dq[NM][2];
          if constexpr (BITS != 16) {
            // this lane's (scale, zero) pairs: v = (its group j) * NC + (m, h); pair v was copied
            // by quad lane v % 4 as that lane's (v / 4)-th pair
            constexpr int NC = NM * 2, V = NC * Tr::GPQ;
            const int j = Tr::GPQ == 2 ? (c >> 1) : 0;
            const uint32_t my_z = zsel[sidx];
#pragma unroll
            for (int m = 0; m < NM; ++m)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int v = j * NC + m * 2 + h;
                const int slot = (g * V + v) * 4;
                const float s = __uint_as_float(lds32(st + Ring<NM>::W_BYTES + slot));
                const uint32_t zw = lds32(st + Ring<NM>::W_BYTES + Ring<NM>::S_BYTES + slot);
                const uint32_t zsw = __shfl_sync(0xffffffffu, my_z, (lane & ~3) | (v & 3));
                const uint32_t zs = (zsw >> (16 * (v >> 2))) & 0xffffu;
                const uint32_t z = zs >= 4u ? zs - 4u : (zw >> (8 * zs)) & 0xffu;
                dq[m][h] = make_dq(s, z);
              }
          }
#pragma unroll
          for (int s = 0; s < Tr::STEPS; ++s) {
            uint32_t b0, b1;
            b_frag<BITS>(xv, s, b0, b1);
#pragma unroll
            for (int m = 0; m < NM; ++m) {
              const uint4 w0 = lds128(st + ((m * 2 + 0) * 32 + lane) * 16);
              const uint4 w1 = lds128(st + ((m * 2 + 1) * 32 + lane) * 16);
              uint32_t glo, ghi, g8lo, g8hi;
              a_frag<BITS>(w0, dq[m][0], s, glo, ghi);
              a_frag<BITS>(w1, dq[m][1], s, g8lo, g8hi);
              if (!ok) glo = ghi = g8lo = g8hi = 0u;
              mma16816(acc[m], glo, g8lo, ghi, g8hi, b0, b1);
            }
          }
        }
        __syncwarp();   // every lane is done with this stage before it is refilled
        if (q % cmax == cmax - 1) {
          // end of tile for every warp: partials -> smem, barrier, reduce in warp order
          const int tile = t0 + q / cmax;
          float* rb = red + (tile_seq & 1) * (kWarps * NM * 128);
#pragma unroll
          for (int m = 0; m < NM; ++m) {
            float* pp = rb + (warp * NM + m) * 128;
            pp[g * 8 + 2 * c] = acc[m][0];
            pp[g * 8 + 2 * c + 1] = acc[m][1];
            pp[(g + 8) * 8 + 2 * c] = acc[m][2];
            pp[(g + 8) * 8 + 2 * c + 1] = acc[m][3];
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;
          }
          __syncthreads();
          if (threadIdx.x < 128) {
            const int tok = threadIdx.x >> 4, r16 = threadIdx.x & 15;
            if (tok < nt) {
              float s0 = 0.f, s1 = 0.f;
#pragma unroll
              for (int w = 0; w < kWarps; ++w) {
                const float* pp = rb + (w * NM) * 128 + r16 * 8 + tok;
                s0 = __fadd_rn(s0, pp[0]);
                if (NM == 2) s1 = __fadd_rn(s1, pp[128]);
              }
              const size_t r = (size_t)(tok0 + tok);
              const int n = tile * 16 + r16;
              if (W13) {
                const float silu = __fdiv_rn(s0, __fadd_rn(1.f, expf(-s0)));
                const __nv_bfloat16 hv = __float2bfloat16_rn(__fmul_rn(silu, s1));
                a.h[r * a.F + n] = *reinterpret_cast<const uint16_t*>(&hv);
              } else {
                a.y_part[((size_t)ks * a.part_rows + r) * a.Hd + n] = s0;
              }
            }
          }
          ++tile_seq;
        }
      }
    }
  }
  cp_wait<0>();
}

template <bool W13>
__global__ void __launch_bounds__(kThreads, 1) k_decode_gemv(const FfnArgs a, int SK, int sliceK) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Alloc A;
  constexpr int NM = W13 ? 2 : 1;
  float* red = reinterpret_cast<float*>(smem);                          // 2 x kWarps x NM x 128
  const uint32_t ring_base = (uint32_t)__cvta_generic_to_shared(smem + 2 * kWarps * NM * 128 * sizeof(float));
  uint4* xs = reinterpret_cast<uint4*>(smem + 2 * kWarps * NM * 128 * sizeof(float) +
                                       (size_t)kWarps * Pipe<W13>::STAGES * Ring<NM>::STAGE);
  const int K = W13 ? a.Hd : a.F;
  const int N = W13 ? a.F : a.Hd;
  const int NT = N / 16;
  if (threadIdx.x == 0) compute_alloc(a, gridDim.x / SK, A);
  __syncthreads();
  if (A.n_act == 0) return;
  const int V = A.units_total * SK;
  for (int v = blockIdx.x; v < V; v += gridDim.x) {
    const int unit = v / SK, ks = v - unit * SK;
    int i = 0;
    while (A.first_unit[i + 1] <= unit) ++i;
    const int e = A.expert[i];
    const int u_e = A.first_unit[i + 1] - A.first_unit[i];
    const int part = unit - A.first_unit[i];
    const int t0 = (int)((long long)part * NT / u_e), t1 = (int)((long long)(part + 1) * NT / u_e);
    const int k0 = ks * sliceK;
    const int kl = min(sliceK, K - k0);
    const int be = a.bits[e];
    const int r_lo = a.expert_off[e], r_hi = a.expert_off[e + 1];
    // residency check (device-side fault -> status word; outputs zeroed)
    bool resident = true;
    const DevExpert& E = a.experts[e];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const int mi = W13 ? m : 2;
      if (be == 16) resident &= E.w[mi] != nullptr;
      else resident &= width_index(be) >= 0 && E.q[width_index(be)][mi].codes != nullptr;
    }
    if (!resident) {
      if (threadIdx.x == 0 && a.status) atomicOr(a.status, (unsigned)DYMOE_STATUS_WIDTH_NOT_RESIDENT);
      for (int r = r_lo; r < r_hi; ++r)
        for (int n = t0 * 16 + threadIdx.x; n < t1 * 16; n += blockDim.x) {
          if (W13) a.h[(size_t)r * a.F + n] = 0;
          else a.y_part[((size_t)ks * a.part_rows + r) * a.Hd + n] = 0.f;
        }
      continue;
    }
    if (t1 <= t0 || kl <= 0) continue;
    for (int tok0 = r_lo; tok0 < r_hi; tok0 += kMaxTok) {
      const int nt = min(kMaxTok, r_hi - tok0);
      int pad;
      switch (be) {
        case 2: pad = WT<2>::PAD; break;
        case 4: pad = WT<4>::PAD; break;
        case 8: pad = WT<8>::PAD; break;
        default: pad = WT<16>::PAD; break;
      }
      const int row_gran = sliceK / 8 + pad;
      // stage x slice: token rows tok0.. (zero rows beyond nt), granule-swizzled
      __syncthreads();  // previous pass's readers are done with xs / red
      const int gran = kl / 8;
      for (int idx = threadIdx.x; idx < kMaxTok * gran; idx += blockDim.x) {
        const int t = idx / gran, gi = idx - t * gran;
        uint4 v4 = make_uint4(0, 0, 0, 0);
        if (t < nt) {
          const int r = tok0 + t;
          const uint16_t* src = W13 ? a.x + (size_t)a.perm_token[r] * a.Hd
                                    : a.h + (size_t)r * a.F;
          v4 = *reinterpret_cast<const uint4*>(src + k0 + gi * 8);
        }
        xs[t * row_gran + x_granule(gi)] = v4;
      }
      __syncthreads();
      switch (be) {
        case 2: run_tiles<W13, 2>(a, e, k0, kl, t0, t1, tok0, nt, ks, xs, row_gran, red, ring_base); break;
        case 4: run_tiles<W13, 4>(a, e, k0, kl, t0, t1, tok0, nt, ks, xs, row_gran, red, ring_base); break;
        case 8: run_tiles<W13, 8>(a, e, k0, kl, t0, t1, tok0, nt, ks, xs, row_gran, red, ring_base); break;
        default: run_tiles<W13, 16>(a, e, k0, kl, t0, t1, tok0, nt, ks, xs, row_gran, red, ring_base); break;
      }
    }
  }
}

size_t smem_bytes(bool w13, int sliceK) {
  const int NM = w13 ? 2 : 1;
  const size_t ring = w13 ? (size_t)kWarps * Pipe<true>::STAGES * Ring<2>::STAGE
                          : (size_t)kWarps * Pipe<false>::STAGES * Ring<1>::STAGE;
  return 2 * kWarps * NM * 128 * sizeof(float) + ring + (size_t)kMaxTok * (sliceK / 8 + 4) * 16;
}

}  // namespace

int decode_w2_slices(int F) {
  // K = F split into slices of a multiple of 512 whose x tile (8 tokens) fits 64 KB
  const int max_slice = 4096;
  return (F + max_slice - 1) / max_slice;
}
int decode_w2_slice_k(int F) {
  const int sk = decode_w2_slices(F);
  const int per = (F + sk - 1) / sk;
  return (per + 511) / 512 * 512;
}

cudaError_t launch_ffn_decode(const FfnArgs& a, cudaStream_t s, void* const* ev) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms;
  record_ev(ev, 0, s);
  {
    const size_t sm = smem_bytes(true, a.Hd);
    cudaFuncSetAttribute(k_decode_gemv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_decode_gemv<true><<<grid, kThreads, sm, s>>>(a, 1, a.Hd);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  record_ev(ev, 1, s);
  {
    const int SK = decode_w2_slices(a.F), sliceK = decode_w2_slice_k(a.F);
    const size_t sm = smem_bytes(false, sliceK);
    cudaFuncSetAttribute(k_decode_gemv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int g2 = grid / SK * SK;
    k_decode_gemv<false><<<g2 > 0 ? g2 : SK, kThreads, sm, s>>>(a, SK, sliceK);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  record_ev(ev, 2, s);
  return cudaSuccess;
}

}  // namespace dymoe
