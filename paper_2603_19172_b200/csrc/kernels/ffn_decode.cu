// Decode expert FFN (row a7): fused-dequant SwiGLU GEMV for few tokens per expert, sm_100a.
//
// Paper: P:203 step 4 (executor on a unified mixed-precision weight set), P:312 (Int4/Int2
// experts, skip), P:356 (decode is dominated by fetching expert weights).  Readings D13, D17,
// D18, O6: A = x·deq(W1)^T, B = x·deq(W3)^T in fp32, h = RNE_bf16(silu(A)·B),
// y = h·deq(W2)^T in fp32, deq = RNE_bf16((q - z)·RNE_bf16(s)).
//
// Roofline: HBM.  Every active expert's packed W1/W3/W2 is streamed once per 8-token chunk
// (3·Hd·F·(b/8 + 4/128) bytes per expert).
//
// Arithmetic (issue slots, not bytes, are the limit at Int4/Int2):
//  * multiply-adds on the tensor cores: mma.sync m16n8k16, 16 weight rows as A, the (<= 8)
//    tokens as the N = 8 columns of B, fp32 accumulation;
//  * dequant in registers straight into A fragments (ffn_decode_common.cuh a_frag): Int4/Int2
//    codes OR-ed into a bf16 mantissa (exact 2^e + q), HSUB2 of 2^e + z (exact q - z), HMUL2 by
//    bf16(s) = RNE((q - z)·s), bit-identical to D17; Int8 via the fp32 magic 2^23 + q;
//  * the dot product is permutation-invariant in k, so A fragments take codes in the order they
//    are extracted and x is permuted to match (PRMT on registers loaded from shared memory).
//
// Work decomposition (one launch per matrix pair, persistent, cost-balanced):
//  * grid = 1 CTA of two 8-warp groups per SM (alternating tiles); each CTA walks "virtual
//    CTAs".  Every CTA computes the same allocation of virtual CTAs to the active experts,
//    proportional to each expert's measured streaming time (width x token chunks), so CTAs of
//    Int8 and Int2 experts finish together.
//  * a virtual CTA = (expert, K-slice, range of 16-row tiles).  The 8 warps of a group split
//    every tile's K round-robin by 128-byte item and reduce the 16x8 partial tiles through shared
//    memory in warp order (deterministic; the last warp to arrive reduces, no barrier).  The
//    tokens' x slice is staged once per virtual CTA in shared memory (x_pos layout below).
//  * each warp streams its weights through its own TMA ring: an item is one 128 x 16 box per
//    matrix (128 bytes of each of 16 rows, 128-byte swizzled) plus one box of the group-major
//    dequant words; lane 0 issues, the warp waits on the stage mbarrier.
//  * W1/W3 (gate/up): one K-slice (x = 8 x Hd bf16 in smem), SwiGLU applied in the reduction
//    epilogue, h written as bf16.  W2 (down): K = F is split into SK slices, each writes fp32
//    partials y_part[slice]; the combine kernel sums the slices in order.
#include <cstdlib>

#include "ffn_decode_common.cuh"

namespace dymoe {
namespace dec {

// partial-tile reduction buffer per warp and matrix: [tok 8][row 16] floats
constexpr int kRedTile = 8 * 16;

// Optional per-CTA timeline (tools/dec_trace.py builds a separate library with -DDYMOE_DEC_TRACE;
// the product build has no trace code): (event, globaltimer ns) pairs per CTA for the W13 (0) and
// W2 (1) kernels -- 0 start, 1 allocation done, 5 first weight items issued, 6 staging loop done,
// 2 x slice staged (payload: the unit's width and list position), 3 unit's tiles done, 4 end --
// and first-per-launch stamps inside the first unit (0 prime entry, 1 prime return, 2 unit
// decoded, 3 past the pass-start barrier).
#ifdef DYMOE_DEC_TRACE
constexpr int kTrEv = 32;
__device__ unsigned long long g_dec_tr[2][256][2 * kTrEv];
__device__ int g_dec_trn[2][256];
__device__ unsigned long long g_dec_sub[2][256][8];
__device__ __forceinline__ void dec_tr(bool w13, int& n, int ev) {
  if (threadIdx.x == 0 && n < kTrEv && blockIdx.x < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dec_tr[w13 ? 0 : 1][blockIdx.x][2 * n] = ev;
    g_dec_tr[w13 ? 0 : 1][blockIdx.x][2 * n + 1] = t;
    ++n;
    g_dec_trn[w13 ? 0 : 1][blockIdx.x] = n;
    if (ev == 0)
      for (int i = 0; i < 8; ++i) g_dec_sub[w13 ? 0 : 1][blockIdx.x][i] = 0;
  }
}
#define DEC_TR(ev) dec_tr(W13, tr_n, ev)
__device__ __forceinline__ void dec_sub(bool w13, int i) {   // first stamp per launch wins
  if (threadIdx.x == 0 && blockIdx.x < 256 && g_dec_sub[w13 ? 0 : 1][blockIdx.x][i] == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dec_sub[w13 ? 0 : 1][blockIdx.x][i] = t;
  }
}
#define DEC_SUB(i) dec_sub(W13, i)
#else
#define DEC_SUB(i) do {} while (0)
#define DEC_TR(ev) do {} while (0)
#endif

// Shared-memory budget per kernel (one 512-thread CTA per SM, <= 227 KB):
//   codes ring [warp 16][stage S][m][16 rows][128 B]   (1024-aligned: 128-byte swizzle atoms)
//   meta ring  [warp 16][stage S][m][gq <= 4][16 rows] words
//   red        [group 2][buf NB][warp 8][m][tok 8][row 16] floats
//   x          [tok 8][row_gran granules of 16 B]
//   Alloc table, tile sync words, ring mbarriers
template <bool W13>
struct Cfg {
  // two 16-row operand blocks per tile: W13 = the W1 and W3 rows of the same features; W2 = two
  // consecutive 16-row halves of a 32-row tile (4 KB of codes per item in both kernels)
  static constexpr int NM = 2;
  static constexpr int TILE_ROWS = W13 ? 16 : 32;
  static constexpr int S = 2;
  static constexpr int NB = 1;
  static constexpr int BOXES = 1;             // 128-byte boxes per operand block per item
  static constexpr int CODES = NM * BOXES * 2048;
  static constexpr int META = NM * 256;       // [m][gq <= 4][16 rows] words
  static constexpr int RED = 2 * NB * kWarps * NM * kRedTile * 4;
};

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
// x slice loads: the slice is constant for the whole run_tiles call, so the load is a pure function
// of its address (non-volatile: the compiler may schedule it freely)
__device__ __forceinline__ uint4 lds128_const(uint32_t a) {
  uint4 r;
  asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
  return r;
}

__device__ __forceinline__ void mbar_init(uint32_t a, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "DYMOE_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra DYMOE_WAIT_%=;\n}" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(bar) : "memory");
}
// Warp-collective forms: every lane executes them with warp-uniform operands and one elected
// lane (e != 0) issues, so the operands go to uniform registers without a per-lane loop around
// each TMA instruction
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n}" : "=r"(e));
  return e;
}
// The weight stream is read once per step: it is loaded with an L2 evict_first policy so that
// the step's small, re-read data (the kernels' code, the expert table, the routing arrays, x, the
// partials) are not flushed out of L2 by ~1 GB of streamed codes every step -- at kernel start
// every miss on them is a DRAM round trip on the ramp's critical path (tools/dec_trace.py).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma2d_e(uint32_t e, uint32_t dst, const CUtensorMap* m, int x, int y,
                                        uint32_t bar, uint64_t pol) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %6;\n}"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(bar), "r"(e), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma3d_e(uint32_t e, uint32_t dst, const CUtensorMap* m, int x, int y,
                                        int z, uint32_t bar, uint64_t pol) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %6, 0;\n\t"
      "@p cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %7;\n}"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(z), "r"(bar), "r"(e), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_e(uint32_t e, uint32_t a, uint32_t tx) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
               "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}" ::"r"(a), "r"(tx), "r"(e) : "memory");
}
__device__ __forceinline__ void mbar_arrive_e(uint32_t e, uint32_t a) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
               "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(a), "r"(e) : "memory");
}
__device__ __forceinline__ void tma3d(uint32_t dst, const CUtensorMap* m, int x, int y, int z,
                                      uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(z), "r"(bar) : "memory");
}

// Dequant parameters from a metadata word (bf16 scale bits << 16 | zero).
template <int BITS>
__device__ __forceinline__ DQ dq_from_meta(uint32_t w) {
  DQ d;
  d.ss = prmt(w, 0u, 0x3232u);                       // (s, s)
  if constexpr (BITS == 2) {
    const uint32_t zl2 = prmt(w, 0u, 0x4040u);       // (z, z)
    d.zz = zl2 + 0x43004300u;                        // bf16(128 + z)
    d.zz1 = zl2 * 4u + 0x42004200u;                  // bf16(32 + z)
    d.zz2 = zl2 * 16u + 0x41004100u;                 // bf16(8 + z)
  } else {
    d.zz = prmt(w, 0x43u, 0x4040u);                  // (bf16(128 + z), bf16(128 + z))
  }
  d.sf = __uint_as_float(w & 0xffff0000u);
  d.zf = __uint_as_float(prmt(w, 0x4B000000u, 0x7440u));   // 2^23 + z
  return d;
}

// One virtual CTA: expert e, k-slice [k0, k0 + kl), tiles [t0, t1), nt tokens whose x slice is
// staged at shared address xs (x_pos layout, row_gran granules per token).  Outputs: W13 -> bf16
// h at out[tok * ostride + n]; W2 -> fp32 partials at out[tok * ostride + n].  seq: this warp's
// running item count (ring slot / mbarrier parity bookkeeping across calls); returns the new one.
//
// Item p of a tile (p = warp + 8 j) covers the 64-byte chunks [NSUB p, NSUB p + NSUB) of every
// row of the tile's K slice (CK k values each; NSUB = 2 BOXES), one 128 x 16 box per operand
// block (W13: W1 and W3 rows of the tile's 16 features; W2: the two 16-row halves of a 32-row
// tile), plus the metadata boxes of the GQ groups those chunks span.
template <bool W13, int BITS, int WPT>
__device__ __noinline__ uint32_t run_tiles(const CUtensorMap* tm0, const CUtensorMap* tm1,
                                           const CUtensorMap* tmm, int k0,
                                           int kl, int t0, int t1, int nt, void* out, int ostride,
                                           uint32_t xs, int row_gran, float* red,
                                           uint32_t codes_base, uint32_t meta_base,
                                           uint32_t bar_base, int* sync, uint32_t seq,
                                           bool prime_only) {
  using Tr = WT<BITS>;
  using C = Cfg<W13>;
  constexpr int NM = C::NM;
  constexpr int S = C::S;
  constexpr int CK = Tr::CHUNK_K;
  constexpr int BOXES = C::BOXES;
  constexpr int NSUB = 2 * BOXES;                               // 64-byte chunks per item
  constexpr int GQ = BITS == 16 ? 0 : NSUB * CK / DYMOE_GROUP;  // groups per item
  constexpr uint32_t TX = NM * BOXES * 2048 + NM * 64 * GQ;
  // meta words of operand block m start at m * MSTRIDE in the stage: W13's 3-D box packs the two
  // blocks ([m][g][16]); W2's one 32-row box is [g][32 rows], block m = rows 16 m .. 16 m + 15
  constexpr int MSTRIDE = W13 ? GQ * 64 : 64;
  constexpr int MGSTRIDE = W13 ? 16 : 32;   // words per group in the stage
  // WPT = warps sharing a tile (wpt_for below): K split over fewer warps when the slice is short
  constexpr int NSG = 2 * kWarps / WPT;              // subgroups per CTA, on interleaved tiles
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int grp = wid / WPT;                         // subgroup: tiles t0 + grp, + NSG, ...
  const int warp = wid % WPT;                        // warp within the subgroup
  const int g = lane >> 2, c = lane & 3;
  const int nck = (kl + CK - 1) / CK;                // 64-byte chunks per tile row slice
  const int npr = (nck + NSUB - 1) / NSUB;           // items per tile
  const int cmax = (npr + WPT - 1) / WPT;            // per warp (same for all warps)
  const int my_tiles = (t1 - t0 - grp + NSG - 1) / NSG;
  const int n_items = (my_tiles > 0 ? my_tiles : 0) * cmax;
  if (n_items == 0) return seq;
  const uint32_t cring = codes_base + wid * (S * C::CODES);
  const uint32_t mring = meta_base + wid * (S * C::META);
  const uint32_t bars = bar_base + wid * (S * 8);
  red += grp * (C::NB * WPT * NM * kRedTile);
  sync += grp * 4;   // [arrivals buf0, arrivals buf1, generation buf0, generation buf1]

  if (prime_only) DEC_SUB(0);
  // the producer (warp-collective issue, one elected lane): this expert's descriptors at this
  // width, loaded by the caller (W2: both operand blocks come from the W2 matrix)
  const CUtensorMap* tmc[NM] = {tm0, tm1};
  const uint64_t pol = evict_first_policy();
  const int kx0 = k0 * BITS / 8 + warp * (BOXES * 128);   // codes x coordinate (bytes), j = 0
  const int gy0 = k0 / DYMOE_GROUP + warp * GQ;      // meta group coordinate at j = 0
  // item (tile ti, j = jj) into ring position sq
  // warp-collective: all lanes call it with the same arguments, one elected lane issues
  auto issue = [&](uint32_t sq, int ti, int jj) {
    const uint32_t el = elect_one();
    const uint32_t slot = sq % S;
    const uint32_t bar = bars + slot * 8;
    if (warp + WPT * jj >= npr) {   // nothing to load: complete the phase, keep parity in step
      mbar_arrive_e(el, bar);
      return;
    }
    mbar_expect_tx_e(el, bar, TX);
    const uint32_t cs = cring + slot * C::CODES;
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int bx = 0; bx < BOXES; ++bx)
        tma2d_e(el, cs + (m * BOXES + bx) * 2048, tmc[m], kx0 + jj * (WPT * BOXES * 128) + bx * 128,
                ti * C::TILE_ROWS + (W13 ? 0 : m * 16), bar, pol);
    if constexpr (BITS != 16) {
      const uint32_t ms = mring + slot * C::META;
      if constexpr (W13) {
        tma3d_e(el, ms, tmm, ti * 16, gy0 + jj * (WPT * GQ), 0, bar, pol);
      } else {
        tma2d_e(el, ms, tmm, ti * 32, gy0 + jj * (WPT * GQ), bar, pol);   // 32 rows x GQ groups
      }
    }
  };

  float acc[NM][4];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;

  // producer cursor: the next item to issue is j_iss of tile tile_iss.  The first S - 1 items are
  // issued by a separate prime call (prime_only) made before the caller stages x / passes its
  // barrier, so the first weights are in flight while the CTA stages its x slice; the run call
  // only advances the cursor past them.
  int tile_iss = t0 + grp, j_iss = 0;
#pragma unroll
  for (int p = 0; p < S - 1; ++p) {
    if (prime_only && p < n_items) issue(seq + p, tile_iss, j_iss);
    if (++j_iss == cmax) { j_iss = 0; tile_iss += NSG; }
  }
  if (prime_only) {
    DEC_SUB(1);
    return seq;
  }

  // per-lane shared-memory offsets: x (token row g, quad position c, x_pos layout); codes of
  // row 8h + g, granule 4 sub + c, 128-byte swizzled (granule ^ row % 8); meta word of row
  // 8h + g for the group the lane's granule falls in
  const uint32_t xlane = xs + (uint32_t)(g * row_gran + c) * 16;
  uint32_t wofs[2], mofs[NSUB];
#pragma unroll
  for (int sub = 0; sub < 2; ++sub) wofs[sub] = g * 128 + (((sub * 4 + c) ^ g) * 16);
#pragma unroll
  for (int sub = 0; sub < NSUB; ++sub) {
    const int gi = BITS == 16 ? 0 : (sub * CK + c * Tr::CODES) / DYMOE_GROUP;
    mofs[sub] = (gi * MGSTRIDE + g) * 4;
  }
  int tile_seq = 0;
  int tile = t0 + grp, j = 0;      // consumer cursor
  for (int q = 0; q < n_items; ++q) {
    // refill: item q + S - 1 goes into the slot consumed in the previous iteration
    if (q + S - 1 < n_items) issue(seq + q + S - 1, tile_iss, j_iss);
    if (++j_iss == cmax) { j_iss = 0; tile_iss += NSG; }
    const uint32_t sq = seq + q;
    const int p = warp + WPT * j;
    const uint32_t slot = sq % S;
    // every phase is waited on, including the empty items' (arrive-only) phases: no mbarrier
    // phase completes unobserved (compute-sanitizer synccheck), at no cost (already complete)
    mbar_wait(bars + slot * 8, (sq / S) & 1);
    if (p < npr) {
      const uint32_t cs = cring + slot * C::CODES;
      const uint32_t ms = mring + slot * C::META;
#pragma unroll
      for (int sub = 0; sub < NSUB; ++sub) {
        const int ci = NSUB * p + sub;
        if (sub > 0 && ci >= nck) break;
        // x for this chunk: beyond the slice the staged x is zero, so codes past the slice end
        // (the next slice's, or TMA's zero fill past the row end) contribute nothing
        const uint32_t xa = xlane + (uint32_t)ci * (2 * CK);
        DQ dq[NM][2];
        if constexpr (BITS != 16) {
#pragma unroll
          for (int m = 0; m < NM; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              dq[m][h] = dq_from_meta<BITS>(lds32(ms + m * MSTRIDE + h * 32 + mofs[sub]));
        }
        uint4 w[NM][2];
#pragma unroll
        for (int m = 0; m < NM; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            w[m][h] = lds128(cs + (m * BOXES + (sub >> 1)) * 2048 + h * 1024 + wofs[sub & 1]);
        using X = XB<BITS>;
#pragma unroll
        for (int blk = 0; blk < X::NB; ++blk) {
          uint4 xb[X::GPB];
#pragma unroll
          for (int i = 0; i < X::GPB; ++i) xb[i] = lds128_const(xa + (blk * X::GPB + i) * 64);
#pragma unroll
          for (int ss = 0; ss < X::SPB; ++ss) {
            const int s = blk * X::SPB + ss;
            uint32_t b0, b1;
            b_frag<BITS>(xb, ss, b0, b1);
#pragma unroll
            for (int m = 0; m < NM; ++m) {
              uint32_t glo, ghi, g8lo, g8hi;
              a_frag<BITS>(w[m][0], dq[m][0], s, glo, ghi);
              a_frag<BITS>(w[m][1], dq[m][1], s, g8lo, g8hi);
              mma16816(acc[m], glo, g8lo, ghi, g8hi, b0, b1);
            }
          }
        }
      }
    }
    __syncwarp();   // every lane is done with this stage before lane 0 refills it
    if (++j == cmax) {
      // end of tile: partials -> red[buf][warp][m][tok][row16]; the LAST warp of the group to
      // arrive (shared-memory counter) reduces in warp order and applies the epilogue -- no
      // barrier, so warps drift up to NB tiles apart.  Buffer b = tile_seq % NB is reused by
      // tile_seq + NB only after its reduction bumped gen[b].
      j = 0;
      const int b = C::NB == 1 ? 0 : (tile_seq & 1);
      const int gen = C::NB == 1 ? tile_seq : (tile_seq >> 1);
      if (lane == 0)
        while (*reinterpret_cast<volatile int*>(&sync[2 + b]) != gen) {}
      __syncwarp();
      float* rb = red + b * (WPT * NM * kRedTile);
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        float* pp = rb + (warp * NM + m) * kRedTile;
        pp[(2 * c) * 16 + g] = acc[m][0];
        pp[(2 * c + 1) * 16 + g] = acc[m][1];
        pp[(2 * c) * 16 + g + 8] = acc[m][2];
        pp[(2 * c + 1) * 16 + g + 8] = acc[m][3];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;
      }
      __threadfence_block();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(&sync[b], 1);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old == WPT - 1) {
        __threadfence_block();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int o = lane + 32 * i, tok = o >> 4, r16 = o & 15;
          if (tok < nt) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int w = 0; w < WPT; ++w) {
              const float* pp = rb + (w * NM) * kRedTile + o;
              s0 = __fadd_rn(s0, pp[0]);
              if (NM == 2) s1 = __fadd_rn(s1, pp[kRedTile]);
            }
            const int n = tile * C::TILE_ROWS + r16;
            if (W13) {
              // silu(A) * B, fast exp / divide (well inside the FFN tolerance)
              const float silu = __fdividef(s0, 1.f + __expf(-s0));
              const __nv_bfloat16 hv = __float2bfloat16_rn(__fmul_rn(silu, s1));
              reinterpret_cast<__nv_bfloat16*>(out)[(size_t)tok * ostride + n] = hv;
            } else {
              reinterpret_cast<float*>(out)[(size_t)tok * ostride + n] = s0;
              reinterpret_cast<float*>(out)[(size_t)tok * ostride + n + 16] = s1;
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          sync[b] = 0;
          __threadfence_block();
          *reinterpret_cast<volatile int*>(&sync[2 + b]) = gen + 1;
        }
      }
      ++tile_seq;
      tile += NSG;
    }
  }
  return seq + n_items;
}

// Warps sharing a tile (each takes every WPT-th 128-byte item of the tile's K slice and the
// group reduces the partial tiles): 8 at BF16 / Int8, 4 at Int4 / Int2 (whose 512 / 1024-k
// items would otherwise leave each warp 1-2 items per tile), halved (down to 2) while a warp
// would get fewer than `min_items` items per tile -- short K slices (the fine-grained layer's
// K = 2048 / 1408) then keep whole items per warp instead of a cross-warp reduction per item.
constexpr int kDecodeMinItems = 6;   // DYMOE_DECODE_MIN_ITEMS overrides (measurement knob)
__device__ __forceinline__ int items_per_tile(int bits, int kl) {
  const int ck = 4 * (128 / bits);                         // WT<BITS>::CHUNK_K
  return ((kl + ck - 1) / ck + 1) / 2;                     // 2 chunks per item
}
__device__ __forceinline__ int wpt_for(int bits, int kl, int min_items) {
  const int ck = 4 * (128 / bits);                         // WT<BITS>::CHUNK_K
  const int npr = ((kl + ck - 1) / ck + 1) / 2;            // items per tile (2 chunks each)
  int w = (bits == 2 || bits == 4) ? 4 : kWarps;
  while (w > 2 && (npr + w - 1) / w < min_items) w >>= 1;
  return w;
}

// x slice layout in shared memory ("x_pos"): [8 tokens][row_gran granules of 16 B].  Within each
// chunk of CK k values (4 * XU4 granules), the granule lane quad position c reads as its i-th
// (logical granule c * XU4 + i) is stored at position i * 4 + c, so a lane's XU4 loads are 64 B
// apart (immediate offsets) and the 4 lanes of a quad hit 4 consecutive bank groups; row_gran = 4
// (mod 8) puts the other token row of an LDS.128 phase on the other four.
__device__ __forceinline__ int x_logical(int pos, int xu4) {
  const int span = 4 * xu4;
  const int chunk = pos / span, w = pos - chunk * span;
  return chunk * span + (w & 3) * xu4 + (w >> 2);
}
__host__ __device__ inline int x_row_gran(int sliceK) { return (sliceK + 255) / 256 * 32 + 4; }

// dynamic shared-memory carve-up (byte offsets; the base is 1024-aligned)
template <bool W13>
struct Smem {
  static constexpr size_t CODES = (size_t)2 * kWarps * Cfg<W13>::S * Cfg<W13>::CODES;
  static constexpr size_t META = (size_t)2 * kWarps * Cfg<W13>::S * Cfg<W13>::META;
  static constexpr size_t RED = Cfg<W13>::RED;
  static constexpr size_t BARS = (size_t)2 * kWarps * Cfg<W13>::S * 8;
  static constexpr int SYNC_INTS = 64;   // 4 words per tile subgroup, up to 8 subgroups; x2 parts
  static __host__ __device__ size_t x_off() { return CODES + META + RED; }
  static __host__ __device__ size_t tail_off(int sliceK) {
    return x_off() + (size_t)kMaxTok * x_row_gran(sliceK) * 16;
  }
  static __host__ __device__ size_t bytes(int sliceK) {
    return tail_off(sliceK) + BARS + SYNC_INTS * sizeof(int) + sizeof(Alloc);
  }
};

template <bool W13>
__global__ void __launch_bounds__(2 * kThreads, 1) k_decode_gemv(const FfnArgs a, int SK, int sliceK) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using C = Cfg<W13>;
  using L = Smem<W13>;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  if (sbase & 1023) __trap();   // the swizzled TMA boxes need 1024-byte alignment
#ifdef DYMOE_DEC_TRACE
  int tr_n = 0;
#endif
  DEC_TR(0);
  const size_t tail = L::tail_off(sliceK);
  uint64_t* ring_bar = reinterpret_cast<uint64_t*>(smem + tail);
  int* tile_sync = reinterpret_cast<int*>(smem + tail + L::BARS);   // [group][4]
  Alloc& A = *reinterpret_cast<Alloc*>(smem + tail + L::BARS + L::SYNC_INTS * sizeof(int));
  const uint32_t codes_base = sbase;
  const uint32_t meta_base = sbase + (uint32_t)L::CODES;
  float* red = reinterpret_cast<float*>(smem + L::CODES + L::META);
  uint4* xs = reinterpret_cast<uint4*>(smem + L::x_off());
  const uint32_t bar_base = (uint32_t)__cvta_generic_to_shared(ring_bar);
  const int K = W13 ? a.Hd : a.F;
  const int N = W13 ? a.F : a.Hd;
  const int NT = N / C::TILE_ROWS;
  const int row_gran = x_row_gran(sliceK);
  if ((threadIdx.x & 31) == 0) {   // each warp's ring mbarriers (one arrival + tx per phase)
    for (int i = 0; i < C::S; ++i) mbar_init(bar_base + ((threadIdx.x >> 5) * C::S + i) * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
  }
  // the codes ring is free until the first TMA: use it as the allocation scratch
  if (threadIdx.x < 32) compute_alloc(a, gridDim.x / SK, W13, A, *reinterpret_cast<AllocScratch*>(smem));
  uint32_t seq = 0;   // this warp's ring position
  __syncthreads();
  DEC_TR(1);
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
    // one round of independent loads: the expert's row range and this width's descriptors (the
    // width itself and the list came from the allocation's shared-memory table) -- every
    // dependent global round trip here is ~1 us of ramp for the whole CTA (tools/dec_trace.py)
    const int be = A.bits[i];
    const int r_lo = __ldg(a.expert_off + e), r_hi = __ldg(a.expert_off + e + 1);
    const DevExpert& E = a.experts[e];
    const CUtensorMap *tm0, *tm1, *tmm = nullptr;
    bool resident;   // residency check (device-side fault -> status word; outputs zeroed)
    if (be == 16) {
      tm0 = E.tm_w[W13 ? 0 : 2];
      tm1 = E.tm_w[W13 ? 1 : 2];
      resident = E.w[W13 ? 0 : 2] != nullptr && E.w[W13 ? 1 : 2] != nullptr;
    } else {
      const int wi = width_index(be);
      const DevQMat* Q = E.q[wi < 0 ? 0 : wi];
      tm0 = Q[W13 ? 0 : 2].tm_codes;
      tm1 = Q[W13 ? 1 : 2].tm_codes;
      tmm = Q[W13 ? 0 : 2].tm_meta;
      resident = wi >= 0 && Q[W13 ? 0 : 2].codes != nullptr && Q[W13 ? 1 : 2].codes != nullptr &&
                 tmm != nullptr;
    }
    // the TMA unit fetches a descriptor on its first use; fetch them now, while the rest of the
    // unit's setup runs, instead of on the first weight issue
    if (resident && threadIdx.x < 3) {
      const CUtensorMap* pm = threadIdx.x == 0 ? tm0 : threadIdx.x == 1 ? tm1 : tmm;
      if (pm != nullptr) asm volatile("prefetch.tensormap [%0];" ::"l"(pm) : "memory");
    }
    if (!resident) {
      if (threadIdx.x == 0 && a.status) atomicOr(a.status, (unsigned)DYMOE_STATUS_WIDTH_NOT_RESIDENT);
      for (int r = r_lo; r < r_hi; ++r)
        for (int n = t0 * C::TILE_ROWS + threadIdx.x; n < t1 * C::TILE_ROWS; n += blockDim.x) {
          if (W13) a.h[(size_t)r * a.F + n] = 0;
          else a.y_part[((size_t)ks * a.part_rows + r) * a.Hd + n] = 0.f;
        }
      continue;
    }
    if (t1 <= t0 || kl <= 0) continue;
    DEC_SUB(2);
    int xu4;
    switch (be) {
      case 2: xu4 = WT<2>::XU4; break;
      case 4: xu4 = WT<4>::XU4; break;
      case 8: xu4 = WT<8>::XU4; break;
      default: xu4 = WT<16>::XU4; break;
    }
    const int gran = kl / 8;                        // granules of real x
    const int npos = (kl + 255) / 256 * 32;         // staged positions (zero beyond gran)
    // The unit's tiles run in (at most) two parts: the rem = ntl mod NSG tiles that would leave
    // some tile subgroups a round short run FIRST on wider subgroups (up to all 16 warps on one
    // tile, each warp a share of its K items), then the full rounds on the width's own subgroups.
    // With whole tiles dealt round-robin a CTA whose unit has one tile more than a multiple of
    // NSG took a whole extra tile time (~10 us at Int4) while its other subgroups idled -- the
    // per-CTA end-time spread measured by tools/dec_trace.py.
    const int wpt = wpt_for(be, kl, a.min_items);
    const int nsg = 2 * kWarps / wpt;
    const int rem = (t1 - t0) % nsg;
    int wpt_a = wpt;
    if (rem) {
      const int npr = items_per_tile(be, kl);
      wpt_a = 2 * kWarps;
      while (wpt_a > wpt && (wpt_a * rem > 2 * kWarps || wpt_a > npr)) wpt_a >>= 1;
    }
    const int ta1 = wpt_a != wpt ? t0 + rem : t1;   // part A [t0, ta1) on wpt_a, part B [ta1, t1)
    for (int tok0 = r_lo; tok0 < r_hi; tok0 += kMaxTok) {
      const int nt = min(kMaxTok, r_hi - tok0);
      void* out = W13 ? (void*)(a.h + (size_t)tok0 * a.F)
                      : (void*)(a.y_part + ((size_t)ks * a.part_rows + tok0) * a.Hd);
      const int ostride = W13 ? a.F : a.Hd;
      const uint32_t xsa = (uint32_t)__cvta_generic_to_shared(xs);
#define DYMOE_RUN(B, W) seq = run_tiles<W13, B, W>(tm0, tm1, tmm, k0, kl, ra, rb, nt, out, ostride, \
                                                   xsa, row_gran, red, codes_base, meta_base,    \
                                                   bar_base, tsync, seq, prime)
      auto tiles = [&](int w, int ra, int rb, int* tsync, bool prime) {
        switch (be * 32 + w) {
          case 2 * 32 + 16: DYMOE_RUN(2, 16); break;
          case 2 * 32 + 8: DYMOE_RUN(2, 8); break;
          case 2 * 32 + 4: DYMOE_RUN(2, 4); break;
          case 2 * 32 + 2: DYMOE_RUN(2, 2); break;
          case 4 * 32 + 16: DYMOE_RUN(4, 16); break;
          case 4 * 32 + 8: DYMOE_RUN(4, 8); break;
          case 4 * 32 + 4: DYMOE_RUN(4, 4); break;
          case 4 * 32 + 2: DYMOE_RUN(4, 2); break;
          case 8 * 32 + 16: DYMOE_RUN(8, 16); break;
          case 8 * 32 + 8: DYMOE_RUN(8, 8); break;
          case 8 * 32 + 4: DYMOE_RUN(8, 4); break;
          case 8 * 32 + 2: DYMOE_RUN(8, 2); break;
          case 16 * 32 + 16: DYMOE_RUN(16, 16); break;
          case 16 * 32 + 8: DYMOE_RUN(16, 8); break;
          case 16 * 32 + 4: DYMOE_RUN(16, 4); break;
          default: DYMOE_RUN(16, 2); break;
        }
      };
#undef DYMOE_RUN
      __syncthreads();  // the previous pass is done with xs / red / tile_sync
      DEC_SUB(3);
      if (threadIdx.x < L::SYNC_INTS) tile_sync[threadIdx.x] = 0;
      // each warp's first weight item goes out now (its own ring slot, no shared state), so the
      // HBM latency overlaps the x staging below
      tiles(wpt_a, t0, ta1, tile_sync, true);
      DEC_TR(5);
      // stage the x slice of this pass's tokens (zero rows beyond nt), x_pos layout: the row
      // offsets first, then every load of a position for all 8 tokens before any store (16
      // independent loads in flight per thread at Int2 instead of a dependent chain per element)
      {
        const uint16_t* xbase = W13 ? a.x : a.h;
        const size_t xstride = W13 ? a.Hd : a.F;
        const uint16_t* xk = xbase + k0;
        int row[kMaxTok];
#pragma unroll
        for (int t = 0; t < kMaxTok; ++t) row[t] = t < nt ? (W13 ? __ldg(a.perm_token + tok0 + t) : tok0 + t) : 0;
        const uint4 z4 = make_uint4(0, 0, 0, 0);
        for (int pos = threadIdx.x; pos < npos; pos += blockDim.x) {
          const int gl = x_logical(pos, xu4);
          uint4 v[kMaxTok];
          if (be == 2) {   // granule pair (gb, gb + 1), element-interleaved (x_perm)
            const int gb = gl & ~1;
            uint4 ga[kMaxTok], gc[kMaxTok];
#pragma unroll
            for (int t = 0; t < kMaxTok; ++t) {
              const uint4* src = reinterpret_cast<const uint4*>(xk + (size_t)row[t] * xstride + gb * 8);
              ga[t] = t < nt && gb < gran ? __ldg(src) : z4;
              gc[t] = t < nt && gb + 1 < gran ? __ldg(src + 1) : z4;
            }
#pragma unroll
            for (int t = 0; t < kMaxTok; ++t) v[t] = x_perm<2>(ga[t], gc[t], gl & 1);
          } else {
#pragma unroll
            for (int t = 0; t < kMaxTok; ++t)
              v[t] = t < nt && gl < gran ? __ldg(reinterpret_cast<const uint4*>(xk + (size_t)row[t] * xstride + gl * 8)) : z4;
            if (be == 4) {
#pragma unroll
              for (int t = 0; t < kMaxTok; ++t) v[t] = x_perm<4>(v[t], v[t], 0);
            }
          }
#pragma unroll
          for (int t = 0; t < kMaxTok; ++t) xs[t * row_gran + pos] = v[t];
        }
      }
      DEC_TR(6);
      __syncthreads();
      DEC_TR(2 | (be << 8) | (i << 16));
      tiles(wpt_a, t0, ta1, tile_sync, false);
      if (ta1 < t1) {
        tiles(wpt, ta1, t1, tile_sync + 32, true);
        __syncthreads();   // part A's reduction buffers are free
        tiles(wpt, ta1, t1, tile_sync + 32, false);
      }
      DEC_TR(3);
    }
  }
  DEC_TR(4);
}

size_t smem_bytes(bool w13, int sliceK) {
  return w13 ? Smem<true>::bytes(sliceK) : Smem<false>::bytes(sliceK);
}

}  // namespace dec
using namespace dec;

int decode_w2_slice_k(int F) {
  // K = F is split into the fewest slices of <= 4096 (x slice of 8 tokens <= 64 KB of shared
  // memory), equal up to a multiple of 512: long slices keep all 8 warps of a group busy even at
  // Int2 (512 k per 128-byte item) and keep the fp32 partial traffic small.
  static const int max_k = [] {   // DYMOE_DECODE_W2_SLICE_MAX overrides (measurement knob)
    const char* v = getenv("DYMOE_DECODE_W2_SLICE_MAX");
    const int m = v ? atoi(v) : 4096;
    return m >= 512 && m <= 4096 ? m : 4096;
  }();
  const int sk = (F + max_k - 1) / max_k;
  const int per = (F + sk - 1) / sk;
  return (per + 511) / 512 * 512;
}
int decode_w2_slices(int F) {
  const int sl = decode_w2_slice_k(F);
  return (F + sl - 1) / sl;
}

cudaError_t launch_ffn_decode(const FfnArgs& args, cudaStream_t s, void* const* ev) {
  // one-time setup, thread-safe (C++11 magic static): several host threads may launch the first
  // layer step concurrently (expert-parallel ranks simulated by threads)
  struct Setup { int sms, dyn_max13, dyn_max2; };
  static const Setup setup = [] {
    Setup r{};
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&r.sms, cudaDevAttrMultiProcessorCount, dev);
    // opt in to the maximum once (227 KB per block); the per-launch size is what each launch
    // requests
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa13{}, fa2{};
    cudaFuncGetAttributes(&fa13, k_decode_gemv<true>);
    cudaFuncGetAttributes(&fa2, k_decode_gemv<false>);
    r.dyn_max13 = optin - (int)fa13.sharedSizeBytes;
    r.dyn_max2 = optin - (int)fa2.sharedSizeBytes;
    cudaFuncSetAttribute(k_decode_gemv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, r.dyn_max13);
    cudaFuncSetAttribute(k_decode_gemv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, r.dyn_max2);
    return r;
  }();
  const int sms = setup.sms, dyn_max13 = setup.dyn_max13, dyn_max2 = setup.dyn_max2;
  static const int min_items = [] {
    const char* v = getenv("DYMOE_DECODE_MIN_ITEMS");
    return v ? atoi(v) : kDecodeMinItems;
  }();
  FfnArgs a = args;
  a.min_items = min_items;
  const int SK = decode_w2_slices(a.F), sliceK = decode_w2_slice_k(a.F);
  const size_t sm13 = smem_bytes(true, a.Hd), sm2 = smem_bytes(false, sliceK);
  if ((int)sm13 > dyn_max13 || (int)sm2 > dyn_max2) return cudaErrorInvalidConfiguration;
  const int grid = sms;   // one 512-thread CTA (two 8-warp groups) per SM
  record_ev(ev, 0, s);
  k_decode_gemv<true><<<grid, 2 * kThreads, sm13, s>>>(a, 1, a.Hd);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  record_ev(ev, 1, s);
  const int g2 = grid / SK * SK;
  k_decode_gemv<false><<<g2 > 0 ? g2 : SK, 2 * kThreads, sm2, s>>>(a, SK, sliceK);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  record_ev(ev, 2, s);
  return cudaSuccess;
}

#ifdef DYMOE_DEC_TRACE
extern "C" int dymoe_dec_trace_read(unsigned long long* host, int* counts) {
  static int zero[2][256];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(counts, dec::g_dec_trn, sizeof(zero));
  cudaMemcpyFromSymbol(host, dec::g_dec_tr, sizeof(dec::g_dec_tr));
  cudaMemcpyToSymbol(dec::g_dec_trn, zero, sizeof(zero));
  cudaMemcpyFromSymbol(host + sizeof(dec::g_dec_tr) / 8, dec::g_dec_sub, sizeof(dec::g_dec_sub));
  return (int)cudaGetLastError();
}
#endif

cudaError_t preload_ffn_decode() {
  return preload_kernels(dec::k_decode_gemv<true>, dec::k_decode_gemv<false>);
}

}  // namespace dymoe
