// Prefill expert FFN (row a6): fused-dequant grouped GEMM on the 5th-generation tensor cores
// (tcgen05 / TMEM), CTA pairs (cta_group::2), for sm_100a.
//
// Paper: P:203 step 4 (executor on a unified mixed-precision weight set), P:312 (Int4/Int2,
// skip), P:354 (prefill time).  Readings D13, D17, D18, O6: A = xp·deq(W1)^T, B = xp·deq(W3)^T
// (fp32 accumulation in TMEM), h = RNE_bf16(silu(A)·B), y = h·deq(W2)^T (fp32),
// deq = RNE_bf16((q - z)·RNE_bf16(s)).
//
// Roofline: tensor cores (a dense contraction: 2*3*Hd*F flops per routed (token, expert) pair,
// arithmetic intensity 512-3500 flop/B).  Design:
//  * a cluster of 2 CTAs (one TPC) computes a 256-token x 256-column tile with
//    tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16): CTA r holds token rows [128r, 128r+128)
//    of A and B rows [128r, 128r+128) of the tile in its own shared memory, and its TMEM holds
//    its 128 token rows x all 256 columns.  GEMM 1: B rows 0-127 = W1 rows n0.., 128-255 = the
//    same W3 rows, so each CTA sees gate and up side by side (SwiGLU in its epilogue); GEMM 2:
//    256 consecutive W2 rows.  Each CTA reads only its halves of A and B from shared memory
//    (the pair exchanges operands in the tensor core), halving shared-memory traffic per flop
//    against one CTA computing the same tile with two M = 128 MMAs.
//  * warp roles per CTA (14 warps): warp 0 issues the A-tile TMA (128 expert-ordered token rows
//    x 64 k, 128-byte swizzled; BF16 experts: the B tile too); warp 1 allocates TMEM (both CTAs)
//    and, in the leader CTA only, one thread issues the MMAs and tcgen05.commit (multicast to
//    both CTAs' barriers); warps 2-9 dequantize (two threads per B row, 32 k each per stage;
//    packed codes + dequant word streamed 8 stages ahead by per-thread cp.async into a private
//    smem ring; natural-k-order LOP3/PRMT extraction; HSUB2/HMUL2 = D17; st.shared into the
//    swizzled tile; fence.proxy.async; release-arrive on the leader's barrier); warps 10-13 drain
//    TMEM for the epilogue.  TMEM holds two 256-column accumulators, so the epilogue of tile i
//    overlaps the main loop of tile i + 1.
//  * 4-stage pipeline of 32 KB per CTA (A 16 KB + B 16 KB); the leader's full barrier collects
//    both CTAs' TMA bytes (cta_group::2 TMA signals the leader) and both CTAs' producer arrivals.
//  * persistent grid: CTA pair c walks the (expert, 256-token tile, 256-column tile) list with
//    stride (number of pairs).
#include <cstdlib>

#include "../dymoe_internal.cuh"

namespace dymoe {
namespace pf {

constexpr int BM = 128;           // token rows per CTA (UMMA M = 2 * BM across the pair)
constexpr int TOK = 2 * BM;       // tokens per pair tile
constexpr int BNH = 128;          // B rows per CTA (UMMA N = 2 * BNH)
constexpr int NCOL = 2 * BNH;     // TMEM columns per accumulator
constexpr int BK = 64;            // k per stage (one 128-byte swizzle atom row)
constexpr int ROWB = BK * 2;      // bytes per tile row (K-major)
constexpr int KPER = BK / 2;      // k per B-producer thread per stage (two threads per row)
constexpr int STAGES = 5;
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int B_BYTES = BNH * BK * 2;           // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int kBWarps = 8, kEpiWarps = 4;
constexpr int kBWarp0 = 2, kEpiWarp0 = kBWarp0 + kBWarps;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;   // 448
constexpr int PF = 6;                       // raw ring slots (stages of packed codes in flight)
constexpr int RAW_CODES = 128 * 64;         // per slot: 128 B rows x up to 64 bytes (Int8)
constexpr int RAW_SLOT = RAW_CODES + 1024;  // + the 128 rows' dequant words (512 B), 1 KB aligned
constexpr int RAW_BYTES = PF * RAW_SLOT;
constexpr int kSmem = STAGES * STAGE_BYTES + RAW_BYTES + 1024;   // + alignment slack
constexpr uint32_t TMEM_COLS = 2 * NCOL;                // two accumulators

// Optional timeline of CTA 0 (tools/pf_trace.py builds a separate library with -DDYMOE_PF_TRACE;
// the product build has no trace code): (event, clock64) pairs per role -- 0 MMA issuer,
// 1 producer warp 2 lane 0, 2 A-tile TMA thread -- for the W13 (pass 0) and W2 (pass 1) GEMMs.
#ifdef DYMOE_PF_TRACE
__device__ unsigned long long g_pf_tr[2][3][8192];
__device__ int g_pf_trn[2][3];
#define PF_TR_BEGIN int tr_i = 0
#define PF_TR(role, ev)                                                  \
  do {                                                                   \
    if (blockIdx.x == 0 && tr_i < 4096) {                                \
      g_pf_tr[W13 ? 0 : 1][role][2 * tr_i] = (ev);                       \
      g_pf_tr[W13 ? 0 : 1][role][2 * tr_i + 1] = clock64();              \
      ++tr_i;                                                            \
    }                                                                    \
  } while (0)
#define PF_TR_END(role) \
  do {                  \
    if (blockIdx.x == 0) g_pf_trn[W13 ? 0 : 1][role] = tr_i; \
  } while (0)
#else
#define PF_TR_BEGIN do {} while (0)
#define PF_TR(role, ev) do {} while (0)
#define PF_TR_END(role) do {} while (0)
#endif

// ---------------------------------------------------------------------------------------- PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
// arrive on a barrier given by its shared::cluster address (default .release.cta semantics: the
// data the arrival publishes is consumed by the tensor core through the async proxy, which the
// producers' fence.proxy.async already covers -- cluster-scope release / acquire would cost an
// MEMBAR per arrive and an L1 invalidate per poll)
__device__ __forceinline__ void mbar_arrive_cl(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_cl(uint32_t bar_cl, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cl), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity)
      : "memory");
}
// wait with back-off, for the epilogue warps (idle for most of a tile): their polling would
// otherwise take issue slots from the dequant producers on the same SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}
// 2-D TMA load into this CTA's shared memory, completion signalled on the leader's barrier
__device__ __forceinline__ void tma2d_pair(uint32_t dst, const CUtensorMap* m, int x, int y,
                                           uint32_t bar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(bar_cl) : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_local(uint32_t bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
// 2-D TMA load into this CTA's shared memory, completion on this CTA's barrier
__device__ __forceinline__ void tma2d_local(uint32_t dst, const CUtensorMap* m, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// MMA issue and commit to the barrier at the same offset in both CTAs of the pair, warp-collective:
// every lane executes them with warp-uniform operands and one elected lane issues (no
// per-instruction R2UR / elect loop around a lane-0-only branch)
__device__ __forceinline__ void tc_commit_pair_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
      ::"r"(bar), "h"((uint16_t)0x3) : "memory");
}
__device__ __forceinline__ void tc_mma_pair_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);        // start address
  d |= (uint64_t)1u << 16;                        // leading byte offset (unused when swizzled)
  d |= (uint64_t)((8u * ROWB) >> 4) << 32;        // stride byte offset: 8 rows
  d |= (uint64_t)1u << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2u << 61;                        // layout: SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: bf16 A/B, f32 D, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// byte offset of 16-byte chunk j (k = 8j..8j+7) of row r inside a 128B-swizzled K-major tile
__device__ __forceinline__ uint32_t sw_off(int r, int j) {
  return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4));
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t bf2_sub(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t bf2_mul(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmul2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 r = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}

// ---------------------------------------------------------------------------------------- dequant
// Natural-order bf16 pairs from packed codes; every pair = RNE_bf16((q - z)·s) (D17).
struct DQP {
  uint32_t zz, ss;   // bf16x2 (128 + z, 128 + z) and (s, s)
  float zf;          // Int8: 2^23 + z
};
__device__ __forceinline__ DQP dqp_from_meta(uint32_t m) {
  DQP d;
  d.ss = prmt(m, 0u, 0x3232u);
  const uint32_t zb = 0x4300u | (m & 0xffu);
  d.zz = zb | (zb << 16);
  d.zf = __uint_as_float(0x4B000000u | (m & 0xffu));
  return d;
}
__device__ __forceinline__ uint32_t fin(uint32_t magic_pair, const DQP& d) {
  return bf2_mul(bf2_sub(magic_pair, d.zz), d.ss);
}
// Int4: one word = 8 codes (k0..k7) -> 4 bf16 pairs in k order (one 16-byte chunk)
__device__ __forceinline__ uint4 deq_int4_word(uint32_t w, const DQP& d) {
  const uint32_t e = w & 0x0F0F0F0Fu;          // bytes: n0 n2 n4 n6
  const uint32_t o = (w >> 4) & 0x0F0F0F0Fu;   // bytes: n1 n3 n5 n7
  const uint32_t t0 = prmt(e, o, 0x5140u);     // n0 n1 n2 n3
  const uint32_t t1 = prmt(e, o, 0x7362u);     // n4 n5 n6 n7
  const uint32_t M = 0x43434343u;
  uint4 r;
  r.x = fin(prmt(t0, M, 0x7170u), d);   // (n0, n1): bytes [n0, 43, n1, 43]
  r.y = fin(prmt(t0, M, 0x7372u), d);
  r.z = fin(prmt(t1, M, 0x7170u), d);
  r.w = fin(prmt(t1, M, 0x7372u), d);
  return r;
}
// Int2: one word = 16 codes (k0..k15) -> two 16-byte chunks
__device__ __forceinline__ void deq_int2_word(uint32_t w, const DQP& d, uint4& lo, uint4& hi) {
  const uint32_t b0 = w & 0x03030303u;          // c0 c4 c8  c12
  const uint32_t b1 = (w >> 2) & 0x03030303u;   // c1 c5 c9  c13
  const uint32_t b2 = (w >> 4) & 0x03030303u;   // c2 c6 c10 c14
  const uint32_t b3 = (w >> 6) & 0x03030303u;   // c3 c7 c11 c15
  const uint32_t t0 = prmt(b0, b1, 0x5140u);    // c0 c1 c4 c5
  const uint32_t t1 = prmt(b2, b3, 0x5140u);    // c2 c3 c6 c7
  const uint32_t t2 = prmt(b0, b1, 0x7362u);    // c8 c9 c12 c13
  const uint32_t t3 = prmt(b2, b3, 0x7362u);    // c10 c11 c14 c15
  const uint32_t M = 0x43434343u;
  lo.x = fin(prmt(t0, M, 0x7170u), d);   // c0 c1
  lo.y = fin(prmt(t1, M, 0x7170u), d);   // c2 c3
  lo.z = fin(prmt(t0, M, 0x7372u), d);   // c4 c5
  lo.w = fin(prmt(t1, M, 0x7372u), d);   // c6 c7
  hi.x = fin(prmt(t2, M, 0x7170u), d);   // c8 c9
  hi.y = fin(prmt(t3, M, 0x7170u), d);   // c10 c11
  hi.z = fin(prmt(t2, M, 0x7372u), d);   // c12 c13
  hi.w = fin(prmt(t3, M, 0x7372u), d);   // c14 c15
}
// Int8: two words = 8 codes -> one 16-byte chunk
__device__ __forceinline__ uint32_t deq_int8_pair(uint32_t w, int i, const DQP& d) {
  // the two (2^23 + q) - (2^23 + z) subtractions as one packed FADD2 and the exact bf16x2 pack
  // (|q - z| <= 255 has <= 8 significant bits) as one F2FP: 2 ALU instructions per pair, not 3
  uint64_t a, zz, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(prmt(w, 0x4B000000u, 0x7440u + i)), "r"(prmt(w, 0x4B000000u, 0x7441u + i)));
  asm("mov.b64 %0, {%1, %1};" : "=l"(zz) : "f"(-d.zf));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(zz));
  float d0, d1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(r));
  __nv_bfloat162 p = __floats2bfloat162_rn(d0, d1);
  return bf2_mul(*reinterpret_cast<uint32_t*>(&p), d.ss);
}

// ---------------------------------------------------------------------------------------- B producer
// The packed codes of the CTA's 128 B rows arrive by TMA into a PF-slot ring (one thread issues
// them, PF stages ahead: a 64 k x 128 row box, Int8 64-byte / Int4 32-byte swizzled, plus the
// rows' dequant words of the stage's group).  Two producer threads per B row (k halves of 32)
// read their codes back from the slot, release it (one arrive per warp), dequantize in natural k
// order, store into the 128B-swizzled B tile, fence (generic -> async proxy) and arrive on the
// leader's full barrier.  No producer thread has a memory load in flight at its proxy fence.
// BF16 experts: the B tile comes by TMA (warp 0); the producers only arrive, to keep the count.
template <int BE>
struct RawStage {
  static constexpr int NB = KPER * BE / 8;        // bytes per thread per stage
  static constexpr int NV = (NB + 15) / 16;
  uint4 v[NV];
  uint32_t m;
};

// this thread's codes (row wr, k half khalf) from a raw slot, undoing the TMA swizzle
template <int BE>
__device__ __forceinline__ void read_raw(RawStage<BE>& r, uint32_t slot, int wr, int khalf) {
  if constexpr (BE == 8) {          // 64-byte rows, 64B swizzle: granule g at g ^ ((row >> 1) & 3)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int g = (2 * khalf + i) ^ ((wr >> 1) & 3);
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r.v[i].x), "=r"(r.v[i].y), "=r"(r.v[i].z), "=r"(r.v[i].w)
                   : "r"(slot + wr * 64 + g * 16));
    }
  } else if constexpr (BE == 4) {   // 32-byte rows, 32B swizzle: granule g at g ^ ((row >> 2) & 1)
    const int g = khalf ^ ((wr >> 2) & 1);
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.v[0].x), "=r"(r.v[0].y), "=r"(r.v[0].z), "=r"(r.v[0].w)
                 : "r"(slot + wr * 32 + g * 16));
  } else {                          // 16-byte rows, no swizzle
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.v[0].x), "=r"(r.v[0].y)
                 : "r"(slot + wr * 16 + khalf * 8));
  }
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r.m) : "r"(slot + RAW_CODES + wr * 4));
}

template <int BE>
__device__ __forceinline__ void store_stage(const RawStage<BE>& r, uint32_t dst, int wr, int j0) {
  const DQP d = dqp_from_meta(r.m);
  if constexpr (BE == 4) {
#pragma unroll
    for (int i = 0; i < KPER / 32; ++i) {
      const uint32_t wv[4] = {r.v[i].x, r.v[i].y, r.v[i].z, r.v[i].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 o = deq_int4_word(wv[q], d);
        sts128(dst + sw_off(wr, j0 + 4 * i + q), o.x, o.y, o.z, o.w);
      }
    }
  } else if constexpr (BE == 2) {
    const uint32_t wv[2] = {r.v[0].x, r.v[0].y};
#pragma unroll
    for (int q = 0; q < KPER / 16; ++q) {
      uint4 lo, hi;
      deq_int2_word(wv[q], d, lo, hi);
      sts128(dst + sw_off(wr, j0 + 2 * q), lo.x, lo.y, lo.z, lo.w);
      sts128(dst + sw_off(wr, j0 + 2 * q + 1), hi.x, hi.y, hi.z, hi.w);
    }
  } else {  // 8
#pragma unroll
    for (int i = 0; i < KPER / 16; ++i) {
      const uint4 v = r.v[i];   // 16 codes = two 16-byte output chunks
      sts128(dst + sw_off(wr, j0 + 2 * i), deq_int8_pair(v.x, 0, d), deq_int8_pair(v.x, 2, d),
             deq_int8_pair(v.y, 0, d), deq_int8_pair(v.y, 2, d));
      sts128(dst + sw_off(wr, j0 + 2 * i + 1), deq_int8_pair(v.z, 0, d), deq_int8_pair(v.z, 2, d),
             deq_int8_pair(v.w, 0, d), deq_int8_pair(v.w, 2, d));
    }
  }
}

// One tile's k-blocks [kb0, kb1).  full_cl: shared::cluster address of the leader's full_bar[0]
// (stage s at + 8 s); raw ring position (rslot, rphase) shared with the issuer's order.
template <int BE, bool W13>
__device__ __forceinline__ void produce(int khalf, int wr, int kb0, int kb1, uint32_t sbase,
                                        uint32_t raw_base, uint32_t raw_full0, uint32_t raw_empty0,
                                        uint32_t full_cl, uint32_t empty_bar, int& stage,
                                        uint32_t& phase, int& rslot, uint32_t& rphase, int& tr_i) {
  const int j0 = khalf * (KPER / 8);
  const bool lane0 = (threadIdx.x & 31) == 0;
  const bool tr = threadIdx.x == 64;   // producer warp 2, lane 0
  (void)tr;
  (void)tr_i;
  for (int kb = kb0; kb < kb1; ++kb) {
    if constexpr (BE != 16) {
      RawStage<BE> r;
      if (tr) PF_TR(1, 11);
      mbar_wait(raw_full0 + rslot * 8, rphase);
      if (tr) PF_TR(1, 12);
      read_raw<BE>(r, raw_base + rslot * RAW_SLOT, wr, khalf);
      __syncwarp();
      if (lane0) mbar_arrive_local(raw_empty0 + rslot * 8);
      if (++rslot == PF) { rslot = 0; rphase ^= 1; }
      if (tr) PF_TR(1, 13);
      mbar_wait(empty_bar + stage * 8, phase ^ 1);
      if (tr) PF_TR(1, 14);
      store_stage<BE>(r, sbase + stage * STAGE_BYTES + A_BYTES, wr, j0);
      fence_proxy_async();
    } else {
      mbar_wait(empty_bar + stage * 8, phase ^ 1);
    }
    __syncwarp();   // one release-arrive per warp (the whole warp's writes are fenced)
    if (lane0) mbar_arrive_cl(full_cl + stage * 8);
    if (tr) PF_TR(1, 15);
    if (++stage == STAGES) { stage = 0; phase ^= 1; }
  }
}

// ---------------------------------------------------------------------------------------- tiles
struct Sched {
  int n;                                   // active experts
  int expert[DYMOE_MAX_EXPERTS];
  int first[DYMOE_MAX_EXPERTS + 1];        // prefix of tiles per expert
};
// The schedule's expert table, built by warp 0 (all lanes): kept experts (bits > 0, rows > 0)
// in active-list order with the prefix of their tile counts, ceil(rows / tok) token tiles x
// ntiles_n.  Lanes take contiguous blocks of the list and load them in parallel; two warp scans
// (kept count, tiles) place every entry -- one dependent round trip instead of a serial walk
// over the experts by one thread (tens of microseconds at 64 active experts).
// An expert whose assigned width is not resident (codes / bf16 master or their TMA descriptors
// missing, e.g. a pool slot not yet filled) is left out of the schedule and flagged in the status
// word (include/dymoe.h DYMOE_STATUS_WIDTH_NOT_RESIDENT): its h rows are not written and its
// y_perm rows keep the zeros of the pre-GEMM-2 memset, so the combine adds nothing for it.
__device__ __forceinline__ bool prefill_resident(const FfnArgs& a, int e, bool w13) {
  const int be = a.bits[e];
  const DevExpert& E = a.experts[e];
  bool ok = true;
  for (int m = w13 ? 0 : 2; m < (w13 ? 2 : 3); ++m) {
    if (be == 16) {
      ok &= E.w[m] != nullptr && E.tm_wp[m] != nullptr;
    } else {
      const int wi = width_index(be);
      ok &= wi >= 0 && E.q[wi][m].codes != nullptr && E.q[wi][m].tm_raw != nullptr &&
            E.q[wi][m].tm_rawmeta != nullptr;
    }
  }
  return ok;
}

__device__ void build_sched_warp(const FfnArgs& a, int tok, int ntiles_n, Sched& S, int* n_tiles,
                                 bool w13, int* nr_list, int* nr_count) {
  const int lane = threadIdx.x & 31;
  const int n = a.active_list[0];
  const int per = (n + 31) / 32;
  const int i0 = lane * per, i1 = min(n, i0 + per);
  int kept = 0, tiles = 0;
  for (int i = i0; i < i1; ++i) {
    const int e = a.active_list[1 + i];
    const int n_e = a.expert_off[e + 1] - a.expert_off[e];
    if (a.bits[e] == 0 || n_e == 0) continue;
    if (!prefill_resident(a, e, w13)) {
      if (a.status && blockIdx.x == 0)
        atomicOr(a.status, (unsigned)DYMOE_STATUS_WIDTH_NOT_RESIDENT);
      nr_list[atomicAdd(nr_count, 1)] = e;   // rows left out of the schedule (shared memory)
      continue;
    }
    ++kept;
    tiles += ((n_e + tok - 1) / tok) * ntiles_n;
  }
  int ik = kept, it = tiles;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int vk = __shfl_up_sync(0xffffffffu, ik, o), vt = __shfl_up_sync(0xffffffffu, it, o);
    if (lane >= o) { ik += vk; it += vt; }
  }
  int na = ik - kept, acc = it - tiles;
  for (int i = i0; i < i1; ++i) {   // second pass: the loads hit L1 / L2
    const int e = a.active_list[1 + i];
    const int n_e = a.expert_off[e + 1] - a.expert_off[e];
    if (a.bits[e] == 0 || n_e == 0 || !prefill_resident(a, e, w13)) continue;
    S.expert[na] = e;
    S.first[na] = acc;
    acc += ((n_e + tok - 1) / tok) * ntiles_n;
    ++na;
  }
  if (lane == 31) {
    S.first[na] = acc;
    S.n = na;
    *n_tiles = acc;
  }
}

struct Tile {
  int e, m0, n0, rows;   // expert, first token row (relative), first output column, valid tokens
  int kb0, kb1;          // k-block range of this tile (GEMM 2: one of two K halves)
};
// ntiles_n counts (n tile, k half) pairs when ksplit == 2
// ei: the caller's cursor into the schedule's expert table -- every role walks its tiles in
// increasing t, so the lookup resumes where the previous one stopped (a scan from 0 cost up to
// M shared-memory round trips per tile and role at 64 active experts).
__device__ __forceinline__ Tile tile_at(const Sched& S, const FfnArgs& a, int t, int ntiles_n,
                                        int nstep, int nk, int ksplit, int& ei) {
  int i = ei;
  while (S.first[i + 1] <= t) ++i;
  ei = i;
  Tile r;
  r.e = S.expert[i];
  const int local = t - S.first[i];
  const int n_e = a.expert_off[r.e + 1] - a.expert_off[r.e];
  // column-tile major: consecutive tiles (run concurrently by consecutive clusters) are the
  // expert's token tiles of the SAME weight columns, so a weight tile is streamed from HBM once
  // and served to the other token tiles from L2 (token-tile major re-read every column of the
  // expert's packed weights once per token tile: 2.2x the packed bytes at the Zipf loads)
  const int nmt = (n_e + TOK - 1) / TOK;
  const int ntk = local / nmt, mt = local - ntk * nmt;
  const int nt = ntk / ksplit, kh = ntk - nt * ksplit;
  r.kb0 = (int)((long long)kh * nk / ksplit);
  r.kb1 = (int)((long long)(kh + 1) * nk / ksplit);
  r.m0 = mt * TOK;
  r.n0 = nt * nstep;
  r.rows = min(TOK, n_e - r.m0);
  return r;
}

template <bool W13>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
k_prefill_gemm(const FfnArgs a, const __grid_constant__ CUtensorMap tmA, int ksplit_w2) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Sched S;
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t raw_full[PF], raw_empty[PF];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int n_tiles_sh;
  __shared__ int nr_list[DYMOE_MAX_EXPERTS], nr_count;   // experts left out (width not resident)
  constexpr uint32_t IDESC = make_idesc(2 * BM, NCOL);
  const int K = W13 ? a.Hd : a.F;
  const int NWR = W13 ? a.F : a.Hd;                  // weight rows per matrix
  const int nstep = W13 ? BNH : NCOL;                // output features per tile
  // GEMM 2 (K = F long, only Hd / 256 column tiles per token tile) splits K in two halves whose
  // fp32 partials are added into the zeroed y_perm: exactly two addends per element, so the
  // result does not depend on their order (deterministic).  GEMM 1 is not split (SwiGLU needs the
  // full sums).
  const int KSPLIT = W13 ? 1 : ksplit_w2;
  const int ntiles_n = (NWR + nstep - 1) / nstep * KSPLIT;
  const int nk = K / BK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  auto sA = [&](int s) { return sbase + s * STAGE_BYTES; };
  auto sB = [&](int s) { return sbase + s * STAGE_BYTES + A_BYTES; };
  const uint32_t full0 = smem_u32(&full_bar[0]), empty0 = smem_u32(&empty_bar[0]);
  const uint32_t raw_base = sbase + STAGES * STAGE_BYTES;   // 1 KB aligned slots
  const uint32_t raw_full0 = smem_u32(&raw_full[0]), raw_empty0 = smem_u32(&raw_empty[0]);
  const uint32_t full_cl = mapa(full0, 0);                     // the leader's full barriers
  const uint32_t tempty_cl = mapa(smem_u32(&tempty_bar[0]), 0);

  if (threadIdx.x == 0) nr_count = 0;
  __syncwarp();
  if (threadIdx.x < 32) build_sched_warp(a, TOK, ntiles_n, S, &n_tiles_sh, W13, nr_list, &nr_count);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 2 + 2 * kBWarps);   // leader's: both CTAs arrive
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull_bar[b]), 1);
      mbar_init(smem_u32(&tempty_bar[b]), 2 * kEpiWarps);
    }
    for (int r = 0; r < PF; ++r) {
      mbar_init(smem_u32(&raw_full[r]), 1);         // issuer's expect_tx arrive + TMA bytes
      mbar_init(smem_u32(&raw_empty[r]), kBWarps);  // one arrive per producer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int n_tiles = n_tiles_sh;
  int ei = 0;   // this thread's schedule cursor (tile_at)
  if (!W13 && KSPLIT == 1 && blockIdx.x == 0 && nr_count > 0) {
    // whole-K tiles store y_perm without a pre-zeroed target: the rows of experts left out of
    // the schedule are zeroed here instead, so the combine adds nothing for them (rare path)
    for (int x = 0; x < nr_count; ++x) {
      const int e = nr_list[x];
      const size_t r0 = a.expert_off[e], r1 = a.expert_off[e + 1];
      for (size_t i = r0 * a.Hd + threadIdx.x; i < r1 * a.Hd; i += blockDim.x) a.y_perm[i] = 0.f;
    }
  }

  if (warp == 0) {
    // ------------------------------------------------------------------ A (and BF16 B) TMA
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      PF_TR_BEGIN;
      for (int t = pair; t < n_tiles; t += npairs) {
        const Tile T = tile_at(S, a, t, ntiles_n, nstep, nk, KSPLIT, ei);
        const int row0 = a.expert_off[T.e] + T.m0 + (int)rank * BM;
        const bool bf = a.bits[T.e] == 16;
        const CUtensorMap* tmB = nullptr;
        int brow0 = 0;
        if (bf) {
          const DevExpert& E = a.experts[T.e];
          tmB = E.tm_wp[W13 ? (int)rank : 2];
          brow0 = T.n0 + (W13 ? 0 : (int)rank * BNH);
        }
        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          PF_TR(2, 21);
          mbar_wait(empty0 + stage * 8, phase ^ 1);
          PF_TR(2, 22);
          mbar_expect_tx_cl(full_cl + stage * 8, A_BYTES + (bf ? B_BYTES : 0));
          tma2d_pair(sA(stage), &tmA, kb * BK, row0, full_cl + stage * 8);
          if (bf) tma2d_pair(sB(stage), tmB, kb * BK, brow0, full_cl + stage * 8);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      PF_TR_END(2);
    } else if (lane == 1) {
      // packed codes + dequant words of this CTA's 128 B rows, PF stages ahead of the producers
      int rslot = 0;
      uint32_t rphase = 0;
      for (int t = pair; t < n_tiles; t += npairs) {
        const Tile T = tile_at(S, a, t, ntiles_n, nstep, nk, KSPLIT, ei);
        const int be = a.bits[T.e];
        if (be == 16) continue;
        const DevQMat& q = a.experts[T.e].q[width_index(be)][W13 ? (int)rank : 2];
        const int row0 = T.n0 + (W13 ? 0 : (int)rank * BNH);   // rows past the end: zero fill
        const int rb = BK * be / 8;                              // code bytes per row per stage
        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          mbar_wait(raw_empty0 + rslot * 8, rphase ^ 1);
          mbar_expect_tx_local(raw_full0 + rslot * 8, 128 * rb + 128 * 4);
          tma2d_local(raw_base + rslot * RAW_SLOT, q.tm_raw, kb * rb, row0, raw_full0 + rslot * 8);
          tma2d_local(raw_base + rslot * RAW_SLOT + RAW_CODES, q.tm_rawmeta, row0,
                      kb * BK / DYMOE_GROUP, raw_full0 + rslot * 8);
          if (++rslot == PF) { rslot = 0; rphase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader)
    // The whole warp runs the loop (warp-uniform control flow and descriptors), one elected lane
    // issues.  The waits for the next k-block's stage (and, at a tile change, the next tile's
    // accumulator and schedule lookup) sit before the k-block's last MMA, so that they overlap
    // the MMAs still queued in the tensor core instead of leaving it idle between k-blocks.
    if (rank == 0) {
      int stage = 0, i = 0;
      uint32_t phase = 0;
      int t = pair;
      PF_TR_BEGIN;
      Tile T{};
      if (t < n_tiles) {
        T = tile_at(S, a, t, ntiles_n, nstep, nk, KSPLIT, ei);
        mbar_wait(smem_u32(&tempty_bar[0]), 1);
        mbar_wait(full0, 0);
        tc_fence_after();
      }
      int kb = T.kb0;
      while (t < n_tiles) {
        const int b = i & 1;
        const uint64_t ad = sw_desc(sA(stage)), bd = sw_desc(sB(stage));
        const uint32_t d_tmem = tmem + b * NCOL;
        const uint32_t acc0 = kb != T.kb0;
#pragma unroll
        for (int kk = 0; kk < BK / 16 - 1; ++kk)   // + kk * 32 bytes = + 2 kk in the start field
          tc_mma_pair_elect(d_tmem, ad + 2 * kk, bd + 2 * kk, IDESC, acc0 | (uint32_t)(kk != 0));
        // the next k-block: this tile's, or the first of the next tile
        int nkb = kb + 1, nt = t, ni = i;
        Tile NT = T;
        const bool tile_end = nkb >= T.kb1;
        if (tile_end) {
          nt = t + npairs;
          ni = i + 1;
          if (nt < n_tiles) {
            NT = tile_at(S, a, nt, ntiles_n, nstep, nk, KSPLIT, ei);
            nkb = NT.kb0;
          }
        }
        const int nstage = stage + 1 == STAGES ? 0 : stage + 1;
        const uint32_t nphase = stage + 1 == STAGES ? phase ^ 1 : phase;
        if (lane == 0) PF_TR(0, tile_end ? 5 : 1);
        if (nt < n_tiles) {
          if (tile_end) mbar_wait(smem_u32(&tempty_bar[ni & 1]), ((ni >> 1) & 1) ^ 1);
          if (lane == 0) PF_TR(0, 2);
          mbar_wait(full0 + nstage * 8, nphase);
        }
        if (lane == 0) PF_TR(0, 3);
        tc_mma_pair_elect(d_tmem, ad + 2 * (BK / 16 - 1), bd + 2 * (BK / 16 - 1), IDESC, 1);
        tc_commit_pair_elect(empty0 + stage * 8);
        if (tile_end) tc_commit_pair_elect(smem_u32(&tfull_bar[b]));
        tc_fence_after();   // the next k-block's MMAs are ordered after the waits above
        stage = nstage;
        phase = nphase;
        kb = nkb;
        t = nt;
        i = ni;
        T = NT;
      }
      if (lane == 0) PF_TR_END(0);
    }
  } else if (warp < kEpiWarp0) {
    // ------------------------------------------------------------------ B producer (dequant)
    const int tb = threadIdx.x - kBWarp0 * 32;   // 0..255
    const int wr = tb & (BNH - 1);                // B row within this CTA's half
    const int khalf = tb >> 7;
    int stage = 0, rslot = 0;
    uint32_t phase = 0, rphase = 0;
    int tr_i = 0;
    for (int t = pair; t < n_tiles; t += npairs) {
      const Tile T = tile_at(S, a, t, ntiles_n, nstep, nk, KSPLIT, ei);
      const int be = a.bits[T.e];
#define DYMOE_PRODUCE(B) produce<B, W13>(khalf, wr, T.kb0, T.kb1, sbase, raw_base, raw_full0, \
                                         raw_empty0, full_cl, empty0, stage, phase, rslot, rphase, tr_i)
      switch (be) {
        case 2: DYMOE_PRODUCE(2); break;
        case 4: DYMOE_PRODUCE(4); break;
        case 8: DYMOE_PRODUCE(8); break;
        default: DYMOE_PRODUCE(16); break;
      }
#undef DYMOE_PRODUCE
    }
    if (threadIdx.x == 64) PF_TR_END(1);
  } else {
    // ------------------------------------------------------------------ epilogue (TMEM -> global)
    const int q = warp & 3;                       // TMEM lane quarter this warp may access
    const int trow = q * 32 + lane;               // token row within this CTA's half
    int i = 0;
    for (int t = pair; t < n_tiles; t += npairs, ++i) {
      const Tile T = tile_at(S, a, t, ntiles_n, nstep, nk, KSPLIT, ei);
      const int b = i & 1;
      mbar_wait_sleep(smem_u32(&tfull_bar[b]), (i >> 1) & 1, 256);
      tc_fence_after();
      const int mrow = (int)rank * BM + trow;     // row within the pair tile
      const size_t grow = (size_t)(a.expert_off[T.e] + T.m0 + mrow);
      const bool live = mrow < T.rows;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NCOL);
#pragma unroll 1
      for (int cc = 0; cc < (W13 ? BNH : NCOL) / 32; ++cc) {
        if (W13) {
          uint32_t g[32], u[32];
          tmem_ld32(tbase + cc * 32, g);
          tmem_ld32(tbase + BNH + cc * 32, u);
          tmem_ld_wait();
          if (live) {
            uint32_t hv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float h2[2];
#pragma unroll
              for (int k2 = 0; k2 < 2; ++k2) {
                const float A = __uint_as_float(g[2 * j + k2]), B = __uint_as_float(u[2 * j + k2]);
                h2[k2] = __fmul_rn(__fdividef(A, 1.f + __expf(-A)), B);   // fast silu (fp32)
              }
              hv[j] = pack_bf2(h2[0], h2[1]);
            }
            uint4* dstp = reinterpret_cast<uint4*>(a.h + grow * a.F + T.n0 + cc * 32);
#pragma unroll
            for (int j = 0; j < 4; ++j) dstp[j] = make_uint4(hv[4 * j], hv[4 * j + 1], hv[4 * j + 2], hv[4 * j + 3]);
          }
        } else {
          uint32_t v[32];
          tmem_ld32(tbase + cc * 32, v);
          tmem_ld_wait();
          if (live && T.n0 + cc * 32 < NWR) {   // last W2 tile may overhang Hd (clamped rows)
            float* dstp = a.y_perm + grow * a.Hd + T.n0 + cc * 32;
            if (KSPLIT == 1) {   // the whole K: the element's only write
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<float4*>(dstp + 4 * j) =
                    make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
            } else {
              // one of the two K halves: add into the zeroed output (two addends per element)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dstp + 4 * j),
                             "f"(__uint_as_float(v[4 * j])), "f"(__uint_as_float(v[4 * j + 1])),
                             "f"(__uint_as_float(v[4 * j + 2])), "f"(__uint_as_float(v[4 * j + 3]))
                             : "memory");
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cl(tempty_cl + b * 8);
    }
  }
  tc_fence_before();
  cluster_sync();   // both CTAs done (the peer's TMEM and smem are no longer touched)
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace pf

// GEMM 1's A operand in expert order: xp[r] = x[perm_token[r]] for r < expert_off[M] (the one
// partial pair tile past the routed count is zeroed; `rows` is only the capacity), 16-byte vectors.
__global__ void __launch_bounds__(256) k_gather_perm(const uint4* __restrict__ x, int vpr,
                                                     const int32_t* __restrict__ perm_token,
                                                     const int32_t* __restrict__ count, int rows,
                                                     uint4* __restrict__ xp) {
  const int n = *count;
  const size_t lim = (size_t)min(rows, n + pf::TOK) * vpr;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < lim;
       i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / vpr), c = (int)(i - (size_t)r * vpr);
    xp[i] = r < n ? __ldg(x + (size_t)perm_token[r] * vpr + c) : make_uint4(0, 0, 0, 0);
  }
}

cudaError_t launch_ffn_prefill(const FfnArgs& a, cudaStream_t s, void* const* ev) {
  using namespace pf;
  if (a.Hd % BNH || a.F % BNH || a.Hd % BK || a.F % BK) return cudaErrorInvalidValue;
  static const int sms = [] {   // one-time setup, thread-safe (magic static)
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_prefill_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_prefill_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    return n;
  }();
  const int rows = a.T * a.k;
  uint16_t* xp = reinterpret_cast<uint16_t*>(a.y_part);   // scratch: [T*k][Hd] bf16
  CUtensorMap tm13, tm2;
  if (!encode_tmap_2d(&tm13, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, xp, a.Hd, rows, (uint64_t)a.Hd * 2,
                      BK, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_2d(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.h, a.F, rows, (uint64_t)a.F * 2,
                      BK, BM, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  record_ev(ev, 0, s);
  {
    const int vpr = a.Hd / 8;
    const size_t total = (size_t)rows * vpr;
    const unsigned blocks = (unsigned)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    k_gather_perm<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(a.x), vpr, a.perm_token,
                                         a.expert_off + a.M, rows, reinterpret_cast<uint4*>(xp));
  }
  const int grid = sms / 2 * 2;   // whole CTA pairs, one CTA per SM
  // GEMM 2's K = F split in two halves only when it is long (Mixtral F = 14336: 224 k-blocks,
  // 749 vs 722 TFLOP/s); a short K (the fine-grained layer's F = 1408: 22 k-blocks) keeps whole
  // tiles (W2 269 -> 334 TFLOP/s).  DYMOE_PREFILL_W2_KSPLIT overrides (measurement knob).
  static const int ks_env = getenv("DYMOE_PREFILL_W2_KSPLIT") ? atoi(getenv("DYMOE_PREFILL_W2_KSPLIT")) : 0;
  const int ksplit = ks_env > 0 ? ks_env : (a.F / BK >= 64 ? 2 : 1);
  k_prefill_gemm<true><<<grid, kThreads, kSmem, s>>>(a, tm13, 1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  record_ev(ev, 1, s);
  // split-K target: the routed rows (device count) zeroed, not the whole capacity; whole-K
  // tiles store their rows (and zero those of experts left out) themselves
  if (ksplit != 1) {
    e = launch_zero_rows(a.y_perm, a.Hd, rows, a.expert_off + a.M, s);
    if (e != cudaSuccess) return e;
  }
  k_prefill_gemm<false><<<grid, kThreads, kSmem, s>>>(a, tm2, ksplit == 1 ? 1 : 2);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  record_ev(ev, 2, s);
  return cudaSuccess;
}

#ifdef DYMOE_PF_TRACE
extern "C" int dymoe_pf_trace_read(unsigned long long* host, int* counts) {
  int zero[6] = {0, 0, 0, 0, 0, 0};
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(counts, pf::g_pf_trn, sizeof(zero));
  cudaMemcpyFromSymbol(host, pf::g_pf_tr, sizeof(pf::g_pf_tr));
  cudaMemcpyToSymbol(pf::g_pf_trn, zero, sizeof(zero));
  return (int)cudaGetLastError();
}
#endif

cudaError_t preload_ffn_prefill() {
  return preload_kernels(k_gather_perm, pf::k_prefill_gemm<true>, pf::k_prefill_gemm<false>);
}

}  // namespace dymoe
