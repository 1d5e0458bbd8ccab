// Heavy-hitter attention mass without materializing P (Eq. 1 input,
// P:216-221, reading R1): a[h][j] = sum_{i >= j} softmax_{j' <= i}(scale q_i . k_j')[j].
//
// Two passes over causal 128 x 128 blocks of the score matrix on the 5th-generation tensor cores
// (tcgen05.mma.cta_group::1.kind::f16, M = N = 128, K = d = 128, bf16 -> fp32 in TMEM):
//   pass 1 (row statistics): one work item = (head, 128-query block); S = Q_blk K_blk^T for every
//            key block at or below the diagonal; each epilogue thread owns one query row (one TMEM
//            lane) and keeps m_i = max_j s_ij, l_i = sum_j exp(s_ij - m_i) online; it stores
//            n_i = m_i + log2 l_i (log2 units), so that p_ij = 2^(s_ij - n_i);
//   pass 2 (column sums): one work item = (head, 128-key block); S^T = K_blk Q_blk^T for every
//            query block at or after the diagonal, so that a TMEM lane holds one KEY and its
//            row of 128 queries: each epilogue thread adds 2^(s_ij - n_i) over the
//            queries (ascending, four interleaved fp32 chains per key combined in a fixed order --
//            deterministic) and writes a[h][j].
// Per CTA (persistent, one per SM): one lane of warp kTmaWarp streams the tiles by TMA (the work
// item's A tile once into one of two buffers, B tiles through a 4-stage ring; 128B-swizzled
// K-major, two 64-column boxes per 128 x 128 tile), warp kMmaWarp owns TMEM (four 128-column
// accumulators) and issues the MMAs (one elected lane), warps 0 .. 15 drain TMEM in two groups
// that take alternate blocks (tcgen05.ld 32x32b, each warp one 64-column half of its blocks) and
// do the softmax arithmetic -- the MMAs of the next blocks overlap the exponentials of the
// current ones.  Work items are ordered longest first and dealt out in alternating directions;
// pass 2 is a programmatic dependent launch of pass 1.  (Taking every 4th exponential on the FMA
// pipe with a degree-6 polynomial unloaded the SFU but raised the instruction count 70 % and cost
// 20 %.)  The epilogue is bound by the SFU's ex2 (16 / clock / SM, tools/micro/pipe_rates.cu:
// 1024 cycles per 128 x 128 block) plus the per-block TMEM load and per-item combine latencies.
// Roofline: tensor (2 passes x 2 T^2 d H / 2 causal flops) with the SFU's exp2 alongside.
#include "../dymoe_internal.cuh"

namespace dymoe {
namespace attn {

constexpr int D = 128;            // head dim (= MMA K)
constexpr int BT = 128;           // rows / columns per block (MMA M = N)
constexpr int NST = 4;            // B-tile ring stages
constexpr int NACC = 4;           // TMEM accumulators (128 columns each)
constexpr int CHUNK = BT * 128;   // one 64-column box: 128 rows x 128 bytes
constexpr int TILE = 2 * CHUNK;   // 32 KB
constexpr int kSmem = (2 + NST) * TILE + 1024;   // A double-buffered by item, B ring
constexpr int kEpi = 16;          // epilogue warps: two groups of (four lane quarters x two halves)
constexpr int NQ = 4;             // partials per row combined at the end of an item
constexpr int HC = 32;            // columns per tcgen05.ld chunk
// Warp roles: epilogue warps 0 .. kEpi-1, then the TMA and the TMEM/MMA warps.  The roles that
// gate the pipeline take the HIGHEST warp ids: the SM sub-partition scheduler prefers the highest
// eligible warp id, so with the single-thread TMA / MMA warps below the busy epilogue warps, the
// MMA issue of the next block waited behind the current block's exponentials (CTA-0 timeline,
// tools/attn_trace.py: 860 cycles to issue 8 MMAs, 420 cycles of epilogue wait per block).
constexpr int kTmaWarp = kEpi, kMmaWarp = kEpi + 1;
constexpr int kThreads = (kEpi + 2) * 32;
constexpr uint32_t TMEM_COLS = NACC * BT;   // 512: the whole TMEM (one CTA per SM)
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BT >> 3) << 17) |
                           ((uint32_t)(BT >> 4) << 24);   // kind::f16: bf16 x bf16 -> f32, K-major

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity)
      : "memory");
}
// Wait with a back-off between polls (ns): the spinning try_wait of an idle role competes with
// the tensor core's shared-memory operand reads (measurement knobs: DYMOE_ATTN_SLEEP_*).
#ifndef DYMOE_ATTN_SLEEP_TMA
#define DYMOE_ATTN_SLEEP_TMA 0
#endif
#ifndef DYMOE_ATTN_SLEEP_MMA
#define DYMOE_ATTN_SLEEP_MMA 0
#endif
#ifndef DYMOE_ATTN_SLEEP_EPI
#define DYMOE_ATTN_SLEEP_EPI 0
#endif
template <int NS>
__device__ __forceinline__ void mbar_wait_ns(uint32_t bar, uint32_t parity) {
  if constexpr (NS == 0) {
    mbar_wait(bar, parity);
  } else {
    uint32_t done = 0;
    while (true) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done) : "r"(bar), "r"(parity) : "memory");
      if (done) break;
      __nanosleep(NS);
    }
  }
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// warp-collective forms: every lane executes them, one elected lane issues
__device__ __forceinline__ void tc_mma_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(IDESC), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
// K-major, 128-byte swizzle, 8-row atoms 1024 B apart (rows of 128 bytes)
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t (&r)[32] = reinterpret_cast<uint32_t(&)[32]>(v);
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
__device__ __forceinline__ float ex2(float x) {   // 2^x on the SFU (ex2(-inf) = +0)
#ifdef DYMOE_ATTN_FAKE_EX2   // timing experiment only (wrong results): no SFU work
  return __fmaf_rn(x, 0.5f, 1.f);
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}
// Packed fp32 pairs (sm_100 FFMA2 / FADD2): each lane of the pair is the scalar fma.rn / add.rn,
// so the results are bit-identical to the scalar chains with half the FMA-pipe instructions.
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t ex2x2(uint64_t x) {   // (2^x0, 2^x1)
  float a, b;
  upk2(x, a, b);
  return pk2(ex2(a), ex2(b));
}
// Named barriers over the kEpi epilogue warps (barrier 0 is __syncthreads): the item-end partials
// are double-buffered by item parity pb; the writers arrive on "full" barrier 1 + pb and the
// combining warps wait on it, the combining warps arrive on "free" barrier 3 + pb after reading
// and the writers wait on it before they reuse the buffer two items later -- so only the four
// combining warps wait for the slowest warp of an item (a full-CTA barrier around the combine
// held every epilogue warp ~1500 cycles per item).
__device__ __forceinline__ void bar_sync_n(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kEpi * 32) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(kEpi * 32) : "memory");
}

// Work item n (longest first) -> (head, block of the A operand, first and end B block).
// Pass 1: A = query block qb, B = key blocks 0 .. qb.  Pass 2: A = key block kb, B = query
// blocks kb .. nb - 1.
template <bool COLS>
__device__ __forceinline__ void item_at(int n, int H, int nb, int& h, int& a, int& b0, int& b1) {
  const int r = n / H;   // rank in the cost order
  h = n - r * H;
  if (COLS) { a = r; b0 = r; b1 = nb; }
  else { a = nb - 1 - r; b0 = 0; b1 = a + 1; }
}

// The work item of round j for CTA c of G: the rounds alternate direction (round 0: c, round 1:
// 2G-1-c, ...), so a CTA that took a long item in one round takes a short one in the next
// (items are ordered longest first).
__device__ __forceinline__ int snake(int j, int c, int G) { return j * G + ((j & 1) ? G - 1 - c : c); }

// Optional per-role timeline of CTA 0 (tools/attn_trace.py builds a separate library with
// -DDYMOE_ATTN_TRACE; the product build has no trace code): (event, clock64) pairs per role
// (0 MMA issuer, 1 epilogue warp 2, 2 epilogue warp 17).
#ifdef DYMOE_ATTN_TRACE
__device__ unsigned long long g_attn_tr[6][4096];   // roles 0-2: pass 2, 3-5: pass 1
__device__ int g_attn_trn[6];
// the running index lives in a register of the recording thread (`tr_i`, declared by DYMOE_TR_BEGIN)
// so that recording costs two fire-and-forget stores, no load
__device__ unsigned long long g_attn_cta[2][160][3];   // per CTA: entry, work start, end (ns)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DYMOE_TR_BEGIN int tr_i = 0
#define DYMOE_TR(role, ev)                                        \
  do {                                                            \
    if (blockIdx.x == 0 && tr_i < 2048) {                         \
      g_attn_tr[(role) + (COLS ? 0 : 3)][2 * tr_i] = (ev);        \
      g_attn_tr[(role) + (COLS ? 0 : 3)][2 * tr_i + 1] = clock64(); \
      ++tr_i;                                                     \
    }                                                             \
  } while (0)
#define DYMOE_TR_END(role) \
  do {                     \
    if (blockIdx.x == 0) g_attn_trn[(role) + (COLS ? 0 : 3)] = tr_i; \
  } while (0)
#else
#define DYMOE_TR_BEGIN do {} while (0)
#define DYMOE_TR(role, ev) do {} while (0)
#define DYMOE_TR_END(role) do {} while (0)
#endif

template <bool COLS>
__global__ void __launch_bounds__(kThreads, 1)
k_attn_mass(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            int H, int T, float scale_log2, float* __restrict__ m_io, float* __restrict__ l_io,
            float* __restrict__ a_out) {
  extern __shared__ uint8_t smem_raw[];
  // Pass 2 is launched as a programmatic dependent of pass 1 (launch_attention_mass): pass 1
  // lets it launch at once, so each SM starts pass 2's prologue, TMA loads and QK^T MMAs as soon
  // as its pass-1 CTA exits; only pass 2's epilogue, which reads pass 1's n_i, waits for the
  // whole of pass 1 (griddepcontrol.wait) -- pass 1's tail and the launch gap overlap pass 2.
  if (!COLS) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef DYMOE_ATTN_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_attn_cta[COLS][blockIdx.x][0] = gtimer();
#endif
  __shared__ __align__(8) uint64_t full_bar[NST], empty_bar[NST], tfull_bar[NACC], tempty_bar[NACC];
  __shared__ __align__(8) uint64_t a_full[2], a_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float x_m[2][NQ][BT], x_l[2][NQ][BT];           // item partials, by item parity
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA0 = smem_u32(smem);
  auto sA = [&](int it) { return sA0 + (uint32_t)(it & 1) * TILE; };
  auto sB = [&](int s) { return sA0 + (uint32_t)(2 + s) * TILE; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = (T + BT - 1) / BT;
  const int n_items = H * nb;
  const CUtensorMap* tmA = COLS ? &tmK : &tmQ;
  const CUtensorMap* tmB = COLS ? &tmQ : &tmK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(smem_u32(&tfull_bar[b]), 1);
      mbar_init(smem_u32(&tempty_bar[b]), kEpi / 2);   // the 8 warps of the block's group
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&a_full[b]), 1);
      mbar_init(smem_u32(&a_empty[b]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
#ifdef DYMOE_ATTN_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_attn_cta[COLS][blockIdx.x][1] = gtimer();
#endif

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0, it = 0;
      uint32_t phase = 0;
      for (int j = 0;; ++j, ++it) {
        const int n = snake(j, blockIdx.x, gridDim.x);
        if (n >= n_items) break;
        int h, ab, b0, b1;
        item_at<COLS>(n, H, nb, h, ab, b0, b1);
        const uint32_t af = smem_u32(&a_full[it & 1]);
        mbar_wait_ns<DYMOE_ATTN_SLEEP_TMA>(smem_u32(&a_empty[it & 1]), ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(af, TILE);
        tma2d(sA(it), tmA, 0, h * T + ab * BT, af);
        tma2d(sA(it) + CHUNK, tmA, 64, h * T + ab * BT, af);
        for (int bb = b0; bb < b1; ++bb) {
          mbar_wait_ns<DYMOE_ATTN_SLEEP_TMA>(smem_u32(&empty_bar[stage]), phase ^ 1);
          mbar_expect_tx(smem_u32(&full_bar[stage]), TILE);
          tma2d(sB(stage), tmB, 0, h * T + bb * BT, smem_u32(&full_bar[stage]));
          tma2d(sB(stage) + CHUNK, tmB, 64, h * T + bb * BT, smem_u32(&full_bar[stage]));
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (warp-uniform control flow and descriptors) and one elected
    // lane issues each tcgen05 instruction.  The waits for the NEXT block's resources (its A
    // buffer at an item change, its TMEM accumulator, its B stage) sit between the 6th and 7th
    // MMA of the current block, so that they overlap the MMAs still queued in the tensor core:
    // a tcgen05.mma issue blocks while the tensor pipe is busy, and with the waits (~100 cycles
    // each even when already complete) and the loop between blocks the tensor core idled ~40 %
    // (CTA-0 timeline without the epilogue: ~890 cycles per block for 512 of MMA work).
    DYMOE_TR_BEGIN;
    if (lane == 0) DYMOE_TR(0, 100 + COLS);
    int j = 0, it = 0, stage = 0, blk = 0;
    uint32_t phase = 0;
    int h, ab, b0, b1;
    bool have = false;
    {
      const int n = snake(0, blockIdx.x, gridDim.x);
      if (n < n_items) {
        item_at<COLS>(n, H, nb, h, ab, b0, b1);
        have = true;
        mbar_wait(smem_u32(&a_full[0]), 0);
        mbar_wait_ns<DYMOE_ATTN_SLEEP_MMA>(smem_u32(&tempty_bar[0]), 1);
        mbar_wait_ns<DYMOE_ATTN_SLEEP_MMA>(smem_u32(&full_bar[0]), 0);
        tc_fence_after();
      }
    }
    int bb = b0;
    while (have) {
      const int b = blk & (NACC - 1);
      const uint64_t adesc = sw_desc(sA(it)), bdesc = sw_desc(sB(stage));
      if (lane == 0) DYMOE_TR(0, 3);
      constexpr int KS = D / 16;   // MMAs per block
#pragma unroll
      for (int kk = 0; kk < KS - 2; ++kk) {
        // + byte offset / 16 in the descriptor's start-address field (no carry out of it:
        // shared addresses < 256 KB)
        const uint32_t off = ((uint32_t)(kk >> 2) * CHUNK + (uint32_t)(kk & 3) * 32) >> 4;
        tc_mma_elect(tmem + (uint32_t)(b * BT), adesc + off, bdesc + off, kk != 0);
      }
      // the next block: same item, or the first block of the next item
      int nj = j, nit = it, nbb = bb + 1, nb1 = b1, nh = h, nab = ab;
      bool nhave = true, new_item = false;
      if (nbb >= b1) {
        nj = j + 1;
        const int n2 = snake(nj, blockIdx.x, gridDim.x);
        if (n2 < n_items) {
          int nb0;
          item_at<COLS>(n2, H, nb, nh, nab, nb0, nb1);
          nbb = nb0;
          nit = it + 1;
          new_item = true;
        } else {
          nhave = false;
        }
      }
      const int nstage = stage + 1 == NST ? 0 : stage + 1;
      const uint32_t nphase = stage + 1 == NST ? phase ^ 1 : phase;
      const int nblk = blk + 1;
      if (nhave) {
        if (lane == 0) DYMOE_TR(0, 1);
        if (new_item) mbar_wait(smem_u32(&a_full[nit & 1]), (nit >> 1) & 1);
        mbar_wait_ns<DYMOE_ATTN_SLEEP_MMA>(smem_u32(&tempty_bar[nblk & (NACC - 1)]),
                                           ((nblk / NACC) & 1) ^ 1);
        mbar_wait_ns<DYMOE_ATTN_SLEEP_MMA>(smem_u32(&full_bar[nstage]), nphase);
        if (lane == 0) DYMOE_TR(0, 2);
      }
#pragma unroll
      for (int kk = KS - 2; kk < KS; ++kk) {
        const uint32_t off = ((uint32_t)(kk >> 2) * CHUNK + (uint32_t)(kk & 3) * 32) >> 4;
        tc_mma_elect(tmem + (uint32_t)(b * BT), adesc + off, bdesc + off, 1);
      }
      tc_commit_elect(smem_u32(&empty_bar[stage]));
      tc_commit_elect(smem_u32(&tfull_bar[b]));
      // every MMA reading this item's A buffer has been issued: release it on their completion
      if (!nhave || new_item) tc_commit_elect(smem_u32(&a_empty[it & 1]));
      if (lane == 0) DYMOE_TR(0, 4);
      tc_fence_after();   // the next block's MMAs are ordered after the waits above
      have = nhave;
      j = nj; it = nit; bb = nbb; b1 = nb1; h = nh; ab = nab;
      stage = nstage; phase = nphase; blk = nblk;
    }
    if (lane == 0) DYMOE_TR_END(0);
  } else {
    // ------------------------------------------------------------------ epilogue (warps 0 .. kEpi-1)
    // Two groups of 8 warps take alternate blocks (group g: the blocks with blk % 2 == g, TMEM
    // accumulators g and g + 2), so that one group's wait for the MMA and tcgen05.ld latency
    // overlap the other group's exponentials: with all 16 warps on every block, the SFU idled
    // ~400 of every ~1650 cycles while the warps of each SM sub-partition waited in step
    // (tools/attn_trace.py).  Within its blocks a warp covers one 64-column half in two chunks of
    // HC = 32 columns (one tcgen05.ld each); each row's reductions run as 4 interleaved chains
    // per warp, combined in a fixed order (chains, then the NQ = 4 (group, half) partials) at the
    // end of the item.  Blocks strictly off the diagonal and inside the sequence take a mask-free
    // path.
    const int q = warp & 3;                    // TMEM lane quarter this warp may access
    const int part = (warp >> 2) & 1;          // 64-column half of the block
    const int grp = warp >> 3;                 // block parity this warp takes
    const int pidx = grp * 2 + part;           // partial slot of the item combine, 0 .. NQ-1
    const int r = q * 32 + lane;               // A row = TMEM lane owned by this thread
    int blk = 0;
    DYMOE_TR_BEGIN;
    if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 100 + COLS);
    if (COLS) asm volatile("griddepcontrol.wait;" ::: "memory");   // pass 1's n_i complete
    int iti = 0;                               // this CTA's item counter
    int n_my = 0;                              // items of this CTA (same walk as the loop below)
    while (snake(n_my, blockIdx.x, gridDim.x) < n_items) ++n_my;
    for (int j = 0;; ++j) {
      const int n = snake(j, blockIdx.x, gridDim.x);
      if (n >= n_items) break;
      int h, ab, b0, b1;
      item_at<COLS>(n, H, nb, h, ab, b0, b1);
      const int row = ab * BT + r;            // query (pass 1) / key (pass 2) of this thread
      float m = -INFINITY, l = 0.f;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int bb = b0; bb < b1; ++bb, ++blk) {
        if ((blk & 1) != grp) continue;
        const int b = blk & (NACC - 1);
        const uint32_t par = (uint32_t)(blk / NACC) & 1;
#ifdef DYMOE_ATTN_NO_EPI   // timing experiment only (wrong results): the MMA pipeline alone
        mbar_wait(smem_u32(&tfull_bar[b]), par);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[b]));
        if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 12);
        continue;
#endif
        const bool full = bb != ab && (bb + 1) * BT <= T;   // no causal / tail mask (uniform)
        const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BT);
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
          const int c0 = part * 2 * HC + ch * HC;
          float s[HC];
          if (COLS) {
            // n_i of this chunk's 32 queries (pass 1): one address per load across the warp (a
            // broadcast from L1), issued before the waits so that their latency overlaps them
            const float* mq = m_io + (size_t)h * T + bb * BT + c0;
            float4 mm4[HC / 4];
            if (full && (T & 3) == 0) {           // 16-byte aligned rows of the scratch
#pragma unroll
              for (int c = 0; c < HC / 4; ++c) mm4[c] = __ldg(reinterpret_cast<const float4*>(mq) + c);
            } else {
              const int nv = min(HC, T - bb * BT - c0);   // queries of this chunk inside the sequence
#pragma unroll
              for (int c = 0; c < HC / 4; ++c) {
                float t0[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) t0[e] = 4 * c + e < nv ? __ldg(mq + 4 * c + e) : 0.f;
                mm4[c] = make_float4(t0[0], t0[1], t0[2], t0[3]);
              }
            }
            if (ch == 0) {
              if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 11);
              mbar_wait_ns<DYMOE_ATTN_SLEEP_EPI>(smem_u32(&tfull_bar[b]), par);
              if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 12);
              tc_fence_after();
            }
            tmem_ld32(tb + c0, s);
            tmem_ld_wait();
            if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 13);
            if (ch == 1) {   // both chunks read: the accumulator may be overwritten
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[b]));
            }
            // queries i = bb*128 + c0 + c; valid when i >= row (causal) and i < T
            if (full) {
              // chains (acc0, acc1) and (acc2, acc3) as packed pairs: the same fma / add per lane
              const uint64_t c2 = pk2(scale_log2, scale_log2);
              uint64_t a01 = pk2(acc[0], acc[1]), a23 = pk2(acc[2], acc[3]);
#pragma unroll
              for (int c = 0; c < HC; c += 4) {
                const float4 mm = mm4[c / 4];
                a01 = fadd2(a01, ex2x2(ffma2(pk2(s[c], s[c + 1]), c2, pk2(-mm.x, -mm.y))));
                a23 = fadd2(a23, ex2x2(ffma2(pk2(s[c + 2], s[c + 3]), c2, pk2(-mm.z, -mm.w))));
              }
              upk2(a01, acc[0], acc[1]);
              upk2(a23, acc[2], acc[3]);
            } else {
              const int cmin = row - bb * BT - c0;   // first valid column of this chunk
              const int cmax = T - bb * BT - c0;     // columns >= cmax are past the sequence
#pragma unroll
              for (int c = 0; c < HC; c += 4) {
                const float4 mm = mm4[c / 4];
                const float mv[4] = {mm.x, mm.y, mm.z, mm.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const bool ok = c + e >= cmin && c + e < cmax;
                  const float p = ex2(__fmaf_rn(s[c + e], scale_log2, -mv[e]));
                  acc[e] += ok ? p : 0.f;
                }
              }
            }
          } else {
            if (ch == 0) {
              if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 11);
              mbar_wait_ns<DYMOE_ATTN_SLEEP_EPI>(smem_u32(&tfull_bar[b]), par);
              if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 12);
              tc_fence_after();
            }
            tmem_ld32(tb + c0, s);
            tmem_ld_wait();
            if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 13);
            if (ch == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[b]));
            }
            // keys j = bb*128 + c0 + c, valid when j <= row (causal) and j < T; the max is taken
            // on the raw scores (scale > 0), the exponent is fma(s, scale_log2, -max * scale_log2)
            if (!full) {
              const int cmax = min(row - bb * BT + 1, T - bb * BT) - c0;
#pragma unroll
              for (int c = 0; c < HC; ++c) s[c] = c < cmax ? s[c] : -INFINITY;
            }
            float bm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int c = 0; c < HC; ++c) bm[c & 3] = fmaxf(bm[c & 3], s[c]);
            const float nm = fmaxf(m, fmaxf(fmaxf(bm[0], bm[1]), fmaxf(bm[2], bm[3])));
            float sum[4] = {0.f, 0.f, 0.f, 0.f};
            if (nm != -INFINITY) {
              const float nms = -nm * scale_log2;
              const uint64_t c2 = pk2(scale_log2, scale_log2), n2 = pk2(nms, nms);
              uint64_t s01 = pk2(0.f, 0.f), s23 = pk2(0.f, 0.f);   // chains (0, 1), (2, 3)
#pragma unroll
              for (int c = 0; c < HC; c += 4) {
                s01 = fadd2(s01, ex2x2(ffma2(pk2(s[c], s[c + 1]), c2, n2)));
                s23 = fadd2(s23, ex2x2(ffma2(pk2(s[c + 2], s[c + 3]), c2, n2)));
              }
              upk2(s01, sum[0], sum[1]);
              upk2(s23, sum[2], sum[3]);
            }
            l = (m == -INFINITY ? 0.f : l * ex2((m - nm) * scale_log2)) +
                ((sum[0] + sum[1]) + (sum[2] + sum[3]));
            m = nm;
          }
        }
      }
      // combine the partials of each row: slots 1.. hand theirs to slot 0
      if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 14);
      const int pb = iti & 1;
      if (pidx != 0 && iti >= 2) bar_sync_n(3 + pb);   // the combine of item iti - 2 has read pb
      x_m[pb][pidx][r] = COLS ? (acc[0] + acc[1]) + (acc[2] + acc[3]) : m;
      x_l[pb][pidx][r] = l;
      if (pidx != 0) {
        bar_arrive_n(1 + pb);
      } else {
        bar_sync_n(1 + pb);
        if (row < T) {
          if (COLS) {
            float a = x_m[pb][0][r];
#pragma unroll
            for (int p = 1; p < NQ; ++p) a += x_m[pb][p][r];
            a_out[(size_t)h * T + row] = a;
          } else {
            float mt = x_m[pb][0][r];   // raw-score maxima; m, l in the scaled log2 domain
#pragma unroll
            for (int p = 1; p < NQ; ++p) mt = fmaxf(mt, x_m[pb][p][r]);
            float lt = 0.f;
#pragma unroll
            for (int p = 0; p < NQ; ++p)
              lt += x_m[pb][p][r] == -INFINITY ? 0.f
                                               : x_l[pb][p][r] * ex2((x_m[pb][p][r] - mt) * scale_log2);
            // p_ij = 2^(s_ij c - m_i) / l_i = 2^(s_ij c - (m_i + log2 l_i)): pass 2 needs one value
            m_io[(size_t)h * T + row] = __fadd_rn(mt * scale_log2, log2f(lt));
            l_io[(size_t)h * T + row] = lt;
          }
        }
        if (iti + 2 < n_my) bar_arrive_n(3 + pb);   // only where a writer will wait for it
      }
      ++iti;
      if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR(warp == 0 ? 1 : 2, 15);
    }
    if (lane == 0 && (warp == 0 || warp == kEpi - 1)) DYMOE_TR_END(warp == 0 ? 1 : 2);
  }
  tc_fence_before();
  __syncthreads();
#ifdef DYMOE_ATTN_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_attn_cta[COLS][blockIdx.x][2] = gtimer();
#endif
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace attn

cudaError_t launch_attention_mass(const uint16_t* Q, const uint16_t* K, int H, int T, int d,
                                  float scale, float* m_scratch, float* l_scratch, float* a_out,
                                  cudaStream_t s) {
  using namespace attn;
  if (d != D) return cudaErrorInvalidValue;
  if (T == 0 || H == 0) return cudaSuccess;
  static const int sms = [] {   // one-time setup, thread-safe (magic static)
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_attn_mass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_attn_mass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    return n;
  }();
  // Q, K as 2-D [H*T][128] bf16 tensors; boxes of 64 columns x 128 rows, 128-byte swizzle (rows
  // of a block past T read the next head's rows or TMA's zero fill: masked in the epilogue)
  CUtensorMap tq, tk;
  const uint64_t rows = (uint64_t)H * T;
  if (!encode_tmap_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Q, D, rows, D * 2, 64, BT,
                      CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_2d(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, D, rows, D * 2, 64, BT,
                      CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const float sl2 = scale * 1.4426950408889634f;
  const int items = H * ((T + BT - 1) / BT);
  const int grid = items < sms ? items : sms;
  k_attn_mass<false><<<grid, kThreads, kSmem, s>>>(tq, tk, H, T, sl2, m_scratch, l_scratch, a_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_attn_mass<true>, tq, tk, H, T, sl2, m_scratch, l_scratch, a_out);
}

#ifdef DYMOE_ATTN_TRACE
extern "C" int dymoe_attn_trace_cta(unsigned long long* host) {   // [2][160][3]
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, attn::g_attn_cta, sizeof(attn::g_attn_cta));
  return (int)cudaGetLastError();
}
extern "C" int dymoe_attn_trace_read(unsigned long long* host, int* counts) {
  int zero[6] = {0, 0, 0, 0, 0, 0};
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(counts, attn::g_attn_trn, sizeof(zero));
  cudaMemcpyFromSymbol(host, attn::g_attn_tr, sizeof(attn::g_attn_tr));
  cudaMemcpyToSymbol(attn::g_attn_trn, zero, sizeof(zero));
  return (int)cudaGetLastError();
}
#endif

cudaError_t preload_attn_mass() {
  return preload_kernels(attn::k_attn_mass<false>, attn::k_attn_mass<true>);
}

}  // namespace dymoe
