/*
 * dymoe.h — C ABI of the B200 (sm_100a) DyMoE mixed-precision MoE layer.
 *
 * Method: "DyMoE: Dynamic Expert Orchestration with Mixed-Precision Quantization for Efficient
 * MoE Inference on Edge" (arxiv 2603.19172).  Citations "P:n" are lines of the paper text
 * (PAPER.md); "Rn"/"Dn" are the readings listed in DESIGN.md §3.
 *
 * Conventions for every entry point
 *  - Tensor arguments are DEVICE pointers owned by the caller (the library never frees them and
 *    keeps none after the call returns), row-major, densely packed, with the shapes stated.
 *    bf16 tensors are passed as uint16_t (IEEE bfloat16 bit patterns).
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream) and
 *    never synchronises the device.  Results are valid once the stream reaches the call.
 *  - Return value: DYMOE_OK or an error code.  On error nothing is launched, and
 *    dymoe_last_error() returns a thread-local message that names the offending argument.
 *  - Inputs must be finite; behaviour on NaN/Inf inputs is undefined.
 *  - Device-side faults that can only be detected while running (e.g. an expert assigned a width
 *    whose packed weights are not resident) set a status word in the workspace, read back by
 *    dymoe_check_status (the only call that synchronises, and only on `stream`).
 */
#ifndef DYMOE_H
#define DYMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dymoe_stream_t; /* identical to cudaStream_t */

enum {
  DYMOE_OK = 0,
  DYMOE_ERR_INVALID = 1,     /* argument validation failed; message names the field */
  DYMOE_ERR_CUDA = 2,        /* a CUDA runtime call or launch failed */
  DYMOE_ERR_NCCL = 3,        /* reserved for collective failures */
  DYMOE_ERR_WORKSPACE = 4,   /* workspace too small or misaligned */
  DYMOE_ERR_UNSUPPORTED = 5, /* shape or width outside what the kernels implement */
  DYMOE_ERR_DEVICE = 6,      /* dymoe_check_status: a device-side fault was recorded */
  DYMOE_ERR_CAPACITY = 7     /* dymoe_pool_insert: the entry cannot fit (nothing changed) */
};

enum { DYMOE_PREFILL = 0, DYMOE_DECODE = 1 };
enum { DYMOE_M_TOTAL = 0, DYMOE_M_ACTIVE = 1 };  /* reading D5: meaning of M in Eq. 5 */
enum { DYMOE_OUT_F32 = 0, DYMOE_OUT_BF16 = 1 };

/* device status word bits (dymoe_check_status) */
enum { DYMOE_STATUS_WIDTH_NOT_RESIDENT = 1 };

#define DYMOE_MAX_TIERS 5
#define DYMOE_MAX_EXPERTS 256
#define DYMOE_GROUP 128          /* quantization group along K (reading D15) */

/* ------------------------------------------------------------------------------------------ */
/* Routing ("the router selects a small subset of experts per token"; gate = Softmax(hW_g),
 * Eq. 6; g_j "the routing weight assigned to expert E_j", Eq. 3).
 *   logits   [T][M] f32  (the gate GEMM is outside the path, reading R19)
 *   topk_idx [T][k] i32  out: experts ordered by (logit desc, index asc); -0.0 == +0.0
 *   topk_w   [T][k] f32  out: softmax over the k selected logits (sums to 1)
 *   probs    [T][M] f32  out, nullable: softmax over all M logits
 * Constraints: T >= 0, 1 <= M <= 256, 1 <= k <= min(M, 8).                                      */
int dymoe_route(const float* logits, int T, int M, int k, int32_t* topk_idx, float* topk_w,
                float* probs, dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Expert importance (PAPER §4.2).
 * PREFILL, token-guided (Eq. 1, Eq. 2):
 *   S_i = sum_{h=0..H-1} attn_mass[h][i] (fp32, head order; R1b), T_imp = the k_tokens tokens
 *   with the largest S (ties: lower index, R11), importance[j] = |{i in T_imp : j in topk_idx[i]}|
 *   stored as exact integers in f32.
 *   attn_mass [H][T] f32; topk_idx [T][k]; k_tokens = 0 means ceil(0.2 T) (R3);
 *   heavy [k_tokens] i32 out, nullable: the members of T_imp in ascending token order;
 *   scratch: device buffer of dymoe_score_scratch_bytes(T) bytes (prefill only, else nullable).
 * DECODE, gate-guided (Eq. 3): logits [B=T][M] f32.
 *   B == 1: importance = the logit row (order-equivalent to g = softmax, exact; D10).
 *   B >  1: importance[j] = sum_b softmax(logits[b])[j], f32, b ascending.
 * importance [M] f32 out.                                                                        */
size_t dymoe_score_scratch_bytes(int T);
int dymoe_score(int phase, const float* attn_mass, int H, const int32_t* topk_idx,
                const float* logits, int T, int M, int k, int k_tokens, float* importance,
                int32_t* heavy, void* scratch, dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Depth-aware precision scheduling (PAPER §4.3): retention r(l) = (1-λ)(cos(π l/(L-1))+1)/2 + λ
 * (Eq. 4; L = 1 gives 1), t = ceil(r(l)·M_eff - 1e-9) (Eq. 5, reading D7),
 * evaluated in fp64.  Tier ladder (reading D9): widths bits[0] > bits[1] > ... > bits[n-1]
 * (each in {16,8,4,2,0}; 0 = skip, "4/0"), thresholds lambdas[0] <= ... <= lambdas[n-2]
 * in [0,1].  Experts ranked by (importance desc, index asc); rank < t_1 -> bits[0],
 * rank < t_2 -> bits[1], ..., else bits[n-1].  clamp_to_k: t_1 >= min(k_route, M_eff) (D8).
 * m_mode TOTAL: M_eff = M; ACTIVE: M_eff = #experts with active_mask != 0, inactive experts
 * get bits[n-1] (D5).  The paper's "4/2" is {bits = {4,2}, lambdas = {λ}}.                    */
typedef struct dymoe_ladder {
  int n_tiers;                         /* 1..5 */
  int bits[DYMOE_MAX_TIERS];
  double lambdas[DYMOE_MAX_TIERS - 1];
  int clamp_to_k;                      /* D8 (default 1) */
  int m_mode;                          /* D5: DYMOE_M_TOTAL or DYMOE_M_ACTIVE */
  int renorm_on_skip;                  /* D12 (used by combine / moe_forward; default 1) */
} dymoe_ladder;

/* importance [M] f32 device; active_mask [M] u8 device (required in ACTIVE mode, else
 * nullable); bits [M] u8 device out; tier_counts [n_tiers-1] host out, nullable — filled
 * only in TOTAL mode (in ACTIVE mode the counts depend on device data).                        */
int dymoe_assign_bits(const float* importance, int M, int layer, int num_layers,
                      const dymoe_ladder* ladder, int k_route, const uint8_t* active_mask,
                      uint8_t* bits, int32_t* tier_counts, dymoe_stream_t stream);

/* Host helper: r(l) of Eq. 4 and the TOTAL-mode tier counts (no device work). */
double dymoe_retention_ratio(int layer, int num_layers, double lambda);
int dymoe_tier_counts(int layer, int num_layers, const dymoe_ladder* ladder, int M_eff,
                      int k_route, int32_t* counts /* [n_tiers-1] */);

/* ------------------------------------------------------------------------------------------ */
/* Group-wise quantization + packing (GPTQ's asymmetric min-max grid as round-to-nearest,
 * readings D14-D16), fp32, exactly in this order per row n and group g of 128 weights along K:
 *   mn = min(0, min w), mx = max(0, max w), s = (mx-mn)/maxq; if s < 2^-126: mn,mx = -1,+1 and
 *   s recomputed (D14b); inv = 1/s; z = rint(-mn*inv); q = clamp(rint(w*inv) + z, 0, maxq)
 *   (rint = half to even, maxq = 2^bits - 1).
 *   W      [N][K] bf16
 *   codes  [N][K*bits/32] u32 out: code k at bits (k % (32/bits))*bits of word k/(32/bits)
 *   scales [N][K/128] f32 out;  zeros [N][K/128] u8 out
 * Constraints: bits in {2,4,8}, group == 128, K % 128 == 0, N >= 0.                           */
int dymoe_quantize(const uint16_t* W, int N, int K, int bits, int group, uint32_t* codes,
                   float* scales, uint8_t* zeros, dymoe_stream_t stream);

typedef struct dymoe_quant_job {
  const uint16_t* W; int N; int K; int bits;
  uint32_t* codes; float* scales; uint8_t* zeros;
} dymoe_quant_job;
/* Many matrices in one launch (e.g. W1/W3/W2 of every expert of a layer). jobs: host array. */
int dymoe_quantize_batched(const dymoe_quant_job* jobs, int n_jobs, int group,
                           dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Expert tables.  A quantized matrix [N][K] at width b (layout of dymoe_quantize): */
typedef struct dymoe_qmat {
  const uint32_t* codes;  /* NULL = this width is not resident */
  const float* scales;
  const uint8_t* zeros;
} dymoe_qmat;

/* One SwiGLU expert (reading D18): W1 (gate) and W3 (up) are [F][Hd], W2 (down) is [Hd][F].
 * w1/w3/w2 are the bf16 masters (needed for the BF16 tier, nullable otherwise);
 * q[wi][m]: width index wi (0 = Int8, 1 = Int4, 2 = Int2), matrix m (0 = W1, 1 = W3, 2 = W2).  */
typedef struct dymoe_expert_desc {
  const uint16_t* w1;
  const uint16_t* w3;
  const uint16_t* w2;
  dymoe_qmat q[3][3];
} dymoe_expert_desc;

typedef struct dymoe_layer_desc {
  int M;         /* experts, 1..256 */
  int k_route;   /* routing top-k, 1..min(M,8) */
  int hidden;    /* Hd, multiple of 128 */
  int ffn;       /* F, multiple of 128 */
  const dymoe_expert_desc* experts;  /* HOST array [M] (its pointers are device pointers) */
} dymoe_layer_desc;

/* Opaque handle holding a device copy of the expert table (created once per layer; the weights
 * themselves stay caller-owned and must outlive the handle).  create synchronises once.
 * The handle also owns a derived per-group word (bf16 bits of RNE_bf16(scale) << 16 | zero) for
 * every resident quantized matrix — the exact pair dequant (D17) consumes — so the decode
 * kernels fetch a group's metadata with one 4-byte copy.  If scales/zeros are re-quantized after
 * create, call dymoe_layer_refresh (asynchronous on `stream`) before the next forward.        */
typedef struct dymoe_layer dymoe_layer;
int dymoe_layer_create(const dymoe_layer_desc* desc, dymoe_layer** out);
int dymoe_layer_refresh(dymoe_layer* layer, dymoe_stream_t stream);
/* Rebind one expert to new formats (pointers as in dymoe_expert_desc; absent widths NULL), e.g.
 * after the expert pool placed or evicted a format.  Rebuilds the expert's derived metadata and
 * TMA descriptors; all device updates are ordered on `stream` before the next forward on it.
 * The previous formats must stay valid until work already queued on other streams is done.    */
int dymoe_layer_set_expert(dymoe_layer* layer, int expert, const dymoe_expert_desc* desc,
                           dymoe_stream_t stream);
int dymoe_layer_destroy(dymoe_layer* layer);

/* ------------------------------------------------------------------------------------------ */
/* Token permutation (P:203 step 3, BASELINE.json "(c)"): the (token, slot) pairs are stably
 * sorted by expert id (ties keep token-major order); pairs routed to an expert with bits == 0
 * (skip, "4/0") are dropped.
 *   topk_idx [T][k] i32; bits [M] u8 device
 *   expert_off [M+1] i32 out: rows of expert e are [expert_off[e], expert_off[e+1])
 *   perm_token, perm_slot [T*k] i32 out (first expert_off[M] valid)
 *   inv_row [T][k] i32 out: row of pair (t, slot) or -1 if dropped
 *   scratch: caller-owned device buffer of dymoe_permute_scratch_bytes(T, k, M) bytes (the
 *   active-expert list and the multi-CTA count/scan arrays); no allocation inside the call.
 * Errors: WORKSPACE if scratch_bytes is too small.                                            */
size_t dymoe_permute_scratch_bytes(int T, int k, int M);
int dymoe_permute(const int32_t* topk_idx, int T, int k, int M, const uint8_t* bits,
                  int32_t* expert_off, int32_t* perm_token, int32_t* perm_slot, int32_t* inv_row,
                  void* scratch, size_t scratch_bytes, dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Expert FFN on the permuted rows (P:203 step 4 "the Model Executor operates on a unified
 * mixed-precision weight set").  For each expert e with bits[e] > 0 and rows r in
 * [expert_off[e], expert_off[e+1]):  A = x[perm_token[r]]·deq(W1_e)^T, B = x[..]·deq(W3_e)^T
 * (fp32 accumulation), h = RNE_bf16(silu(A)*B) (O6), y_perm[r] = h·deq(W2_e)^T (fp32), with
 * deq = RNE_bf16((q - z)·RNE_bf16(s)) (D17) or the bf16 master for bits == 16.
 *   x [T][Hd] bf16; h_ws [T*k][F] bf16 scratch (intermediate); y_perm [T*k][Hd] f32 out.
 * mode: DYMOE_DECODE = fused-dequant GEMV kernels (intended for <= 8 rows per expert),
 *       DYMOE_PREFILL = fused-dequant tcgen05 grouped GEMM.  Both compute the same function.
 * status: device u32 word (nullable) receiving DYMOE_STATUS_* bits.
 * ws: caller-owned device scratch of dymoe_expert_ffn_ws_bytes(layer, T) bytes (256-byte
 *   aligned): the active-expert lists and the decode kernels' W2 K-slice partials / the prefill
 *   kernel's expert-ordered token rows.  No allocation happens inside the call.
 * Errors: WORKSPACE if ws_bytes is too small.                                                  */
size_t dymoe_expert_ffn_ws_bytes(const dymoe_layer* layer, int T);
int dymoe_expert_ffn(const dymoe_layer* layer, int mode, const uint16_t* x, int T,
                     const uint8_t* bits, const int32_t* expert_off, const int32_t* perm_token,
                     uint16_t* h_ws, float* y_perm, uint32_t* status, void* ws, size_t ws_bytes,
                     dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Combine ("0-bit" experts; reading D12): E_t = {slots with inv_row >= 0};
 * w' = topk_w / sum_{E_t} topk_w if renorm else topk_w; y[t] = sum over slots in order of
 * w'·y_perm[inv_row[t][slot]]; E_t empty -> y[t] = 0.  y [T][Hd] f32 or bf16 (out_dtype).     */
int dymoe_combine(const float* y_perm, const int32_t* inv_row, const float* topk_w, int T,
                  int k, int Hd, int renorm, int out_dtype, void* y, dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Mixed-precision expert pool (PAPER.md "Mixed-Precision Cache Management",
 * P:303-309; readings P4-P6).  Host-side policy over a caller-owned arena of
 * `capacity` bytes (typically one device allocation): it decides which (layer, expert) is
 * resident in which format and where, and therefore when dymoe_quantize must run.
 *   Rules (bit widths ordered 16 > 8 > 4 > 2, reading P4): No Duplication (one format per key);
 *   Precision Promotion (request b, narrower cached -> PROMOTE: a miss, load b, evict it);
 *   Conservative Reuse (request b, wider or equal cached -> HIT served by it).  LRU victims.
 *   lookup: outcome DYMOE_POOL_HIT / MISS / PROMOTE, served bits, arena offset (HIT only);
 *     a HIT refreshes recency.
 *   insert: replaces the key's entry (its range freed first; a pinned key -> INVALID), evicts
 *     least-recently-used unpinned entries until a contiguous range fits, places first-fit at
 *     the lowest offset; evicted keys are written as (layer, expert) pairs in eviction order
 *     (at most max_evicted; *n_evicted is the full count).  If the entry cannot fit even with
 *     every unpinned entry evicted: DYMOE_ERR_CAPACITY and nothing changes.
 *   pin / unpin: counted; pinned entries are never evicted.
 *   snapshot: entries least- to most-recently used.  Not thread-safe (one owner thread).      */
typedef struct dymoe_pool dymoe_pool;
enum { DYMOE_POOL_HIT = 0, DYMOE_POOL_MISS = 1, DYMOE_POOL_PROMOTE = 2 };
typedef struct dymoe_pool_entry {
  int layer, expert, bits, pins;
  size_t bytes, offset;
  unsigned long long last_use;
} dymoe_pool_entry;
int dymoe_pool_create(size_t capacity, dymoe_pool** out);
int dymoe_pool_destroy(dymoe_pool* pool);
int dymoe_pool_lookup(dymoe_pool* pool, int layer, int expert, int bits, int* outcome,
                      int* served_bits, size_t* offset);
int dymoe_pool_insert(dymoe_pool* pool, int layer, int expert, int bits, size_t bytes,
                      size_t* offset, int32_t* evicted, int max_evicted, int* n_evicted);
int dymoe_pool_pin(dymoe_pool* pool, int layer, int expert);
int dymoe_pool_unpin(dymoe_pool* pool, int layer, int expert);
int dymoe_pool_snapshot(const dymoe_pool* pool, dymoe_pool_entry* out, int max, int* n);
size_t dymoe_pool_used(const dymoe_pool* pool);

/* Heavy-hitter attention mass (the input of Eq. 1, reading R1) without
 * materializing the attention matrix: a[h][j] = sum_{i >= j} softmax_{j' <= i}(scale *
 * q[h][i] . k[h][j'])[j] (causal).  Two persistent passes of tcgen05 128 x 128 score tiles in
 * TMEM (row max / sum, then column sums of P from K Q^T), fixed summation order.
 *   q, k [H][T][d] bf16 device (d == 128, 16-byte aligned); scale > 0; scratch [2*H*T] f32 device;
 *   a_out [H][T] f32 device (the attn_mass argument of dymoe_score / dymoe_fwd_opts).          */
int dymoe_attention_mass(const uint16_t* q, const uint16_t* k, int H, int T, int d, float scale,
                         float* scratch, float* a_out, dymoe_stream_t stream);

/* Look-ahead prediction of the next layer's experts (PAPER.md "Phase-Adaptive
 * Prefetcher", Eqs. 6-8).  Eq. 6: logits = h · W_g^(l+1)^T evaluated in fp32 with the
 * accuracy of dymoe_gate_logits (below), g_hat = softmax.  PREFILL (Eq. 7): c_e = #{tokens whose top-k_route
 * predicted experts contain e}; requests = the t experts with the largest c_e (> 0), priority =
 * c_e.  DECODE (Eq. 8): requests = top-t of the predicted decode importance (B = 1: the predicted
 * logit row; B > 1: sum over the batch of g_hat), priority = that value.  Order: (value desc,
 * index asc).  The caller uses the requests to stage the next layer's widths (quantize / pool)
 * on a side stream while layer l runs.
 *   h [T][Hd] bf16, w_gate_next [M][Hd] bf16 (Hd multiple of 8, 16-byte aligned), all device.
 *   ws: dymoe_predict_ws_bytes(T, M, k_route) bytes of device scratch.
 *   experts [t] i32 / priority [t] f32 out (first *n_out valid), n_out [1] i32 device out;
 *   logits_out [T][M] f32 (nullable) receives the Eq. 6 logits.
 * Errors: T < 1, M outside [1, 256], k_route outside [1, min(M, 8)], t outside [1, M].        */
size_t dymoe_predict_ws_bytes(int T, int M, int k_route);
int dymoe_predict_next(int phase, const uint16_t* h, const uint16_t* w_gate_next, int T, int Hd,
                       int M, int k_route, int t, void* ws, size_t ws_bytes, int32_t* experts,
                       float* priority, int32_t* n_out, float* logits_out, dymoe_stream_t stream);

/* Router / gate logits (P:111 router; the gate product of Eq. 6, reading P1):
 *   logits[t][e] = h[t] · w_gate[e] + bias[e],
 * the dot product accumulated in fp32 (bf16 x bf16 products are exact in fp32) so that every
 * partial sum passes through at most Hd/32 + 5 roundings, then one fp32 add of bias[e] (bias
 * nullable = 0).  Accuracy contract (reading P1: Eq. 6 fixes the value, not an order):
 *   |logits - exact| <= gamma_(Hd/32+5) · sum_k |h[t][k] w[e][k]|  (+ 2^-24 |logit| with a bias),
 *   gamma_n = n 2^-24 / (1 - n 2^-24); a top-k taken from these logits is therefore the exact
 * top-k wherever the margin exceeds twice that bound.  Deterministic: the same inputs give the
 * same bits on every call.  Used to route each layer of a stack from its own
 * hidden state on the device.
 *   h [T][Hd] bf16, w_gate [M][Hd] bf16 (Hd multiple of 8, 16-byte aligned), bias [M] f32,
 *   logits [T][M] f32 out; all device.
 * Errors: T < 0, M outside [1, 256], Hd not a positive multiple of 8, NULL or misaligned
 * pointers (INVALID).                                                                          */
int dymoe_gate_logits(const uint16_t* h, const uint16_t* w_gate, const float* bias, int T, int Hd,
                      int M, float* logits, dymoe_stream_t stream);

/* RMSNorm of the residual stream before each layer of a stack (the MoE input of a
 * Mixtral block, unit weight for random-init weights):
 *   u[t][i] = RNE_bf16(x[t][i] / sqrt(mean_j x[t][j]^2 + eps)),
 * the mean of squares in fp32 (per-thread sums in order, then fixed-order reductions), one rsqrt.
 *   x, u [T][Hd] bf16 device (16-byte aligned, Hd multiple of 8); u may not alias x.
 * Errors: T < 0, Hd not a positive multiple of 8, eps < 0, NULL / misaligned pointers.          */
int dymoe_rmsnorm(const uint16_t* x, int T, int Hd, float eps, uint16_t* u, dymoe_stream_t stream);

/* Combine weights against the GLOBAL live set (reading D12), for combines that only see part of
 * the slots (expert-parallel decode with the batch replicated on every rank):
 *   w_out[t][s] = bits[topk_idx[t][s]] > 0 ? topk_w[t][s] / d_t : 0,
 *   d_t = sum over live slots in slot order (fp32) if renorm, else 1; no live slot -> 0.
 * Combining a subset of the slots with these weights and renorm = 0 gives exactly the terms
 * dymoe_combine(renorm) would add for those slots.  topk_idx/topk_w/w_out [T][k], bits [M]
 * device; w_out may alias topk_w.                                                              */
int dymoe_renorm_weights(const int32_t* topk_idx, const float* topk_w, const uint8_t* bits, int T,
                         int k, int M, int renorm, float* w_out, dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Expert parallelism (BASELINE.json north_star).  Expert e lives on rank
 * floor(e * P / M) (contiguous blocks).  The owner is non-decreasing in e, so the expert-sorted
 * permutation of dymoe_permute is already ordered by (destination rank, expert, token, slot).
 *   dymoe_ep_plan: send_counts [P] i32 out = rows bound for each rank; row_expert [expert_off[M]]
 *   i32 out = expert of every permuted row.  expert_off [M+1] device.  1 <= P <= min(M, 64).
 *   dymoe_gather_rows: out[i] = x[rows[i]], bf16 rows of Hd (multiple of 8) elements.         */
int dymoe_ep_plan(const int32_t* expert_off, int M, int P, int32_t* send_counts,
                  int32_t* row_expert, dymoe_stream_t stream);
int dymoe_gather_rows(const uint16_t* x, int Hd, const int32_t* rows, int n, uint16_t* out,
                      dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Expert-parallel dispatch and combine over peer memory (the NVLink /
 * NVSwitch replacement of the NCCL all-to-all pair).  Every rank owns one symmetric WINDOW of
 * dymoe_ep_window_bytes(P, M, Hd, cap_rows) device bytes, mapped into every other rank's address
 * space (CUDA IPC between processes; the same pointer between threads of one process):
 *   flags  u32[P]          barrier counters, flags[src] written by rank src
 *   cnt    i32[2][P][M]    cnt[parity][src][e] = rows rank src routes to expert e (double-
 *                          buffered by step parity so a step's publish never races a peer's
 *                          previous combine)
 *   imp    f32[2][P][M]    rank src's local importance (used by dymoe_moe_forward_ep)
 *   red    f32[2][64][Hd]  this rank's partial output (dymoe_moe_forward_ep, replicated decode)
 *   recv_x bf16[cap][Hd]   rows received by this rank, EXPERT-MAJOR: local expert e's rows are
 *                          [Σ_{e'<e} Σ_src cnt[src][e'], ...) and within an expert by source rank,
 *                          then in the source's (token, slot) order -- i.e. exactly the order
 *                          the expert FFN wants, no regrouping on the receiver
 *   y_out  f32[cap][Hd]    the local experts' outputs, row-aligned with recv_x
 * One step (3 barriers):
 *   dymoe_ep_publish_counts   write this rank's per-expert counts (from dymoe_permute's
 *                             expert_off) into cnt[parity][rank][*] of every window
 *   dymoe_ep_barrier
 *   dymoe_ep_dispatch         fused gather + all-to-all: x[perm_token[j]] is stored straight
 *                             into the owner's recv_x row (16-byte stores over NVLink); also
 *                             writes recv_off [M_loc+1] (local expert offsets of recv_x)
 *   dymoe_ep_barrier
 *   dymoe_expert_ffn          on recv_x with recv_off, identity perm, y_perm = the window's y_out
 *   dymoe_ep_barrier
 *   dymoe_ep_combine          fused reverse all-to-all + weighted combine: every live (t, slot)
 *                             pulls its output row from the owner's y_out (NVLink loads) and the
 *                             dymoe_combine arithmetic (reading D12, slot order, fp32) applies.
 * dymoe_ep_window: P ranks, this rank, M experts (expert e on rank floor(e P / M)), Hd, cap_rows
 *   (>= the rows any rank can receive; T_max * k * P is always enough), parity (step & 1) and
 *   peers: a DEVICE array [P] of the windows' base pointers as mapped in this process
 *   (peers[rank] = own window).
 * Barrier: thread p stores `epoch` into flags[rank] of window p (release, system scope), then
 * waits until every flags[src] of its own window is >= epoch (acquire, system scope).  The
 * caller increments epoch by one per barrier call on every rank.  A wait longer than ~5 s sets
 * DYMOE_STATUS_EP_TIMEOUT in *status (nullable) and returns (never hangs the device).
 * Window memory: dymoe_ep_window_alloc (cudaMalloc, zeroed; ipc_handle receives the 64-byte
 * cudaIpcMemHandle_t, nullable), dymoe_ep_window_open (cudaIpcOpenMemHandle with lazy peer
 * access, another process's window), dymoe_ep_window_close / _free.  The caller owns them.
 * Errors: INVALID for NULL pointers, P outside [1, min(M, 64)], rank outside [0, P), Hd not a
 * positive multiple of 8, cap_rows < 0; CUDA for allocation / IPC failures.                   */
enum { DYMOE_STATUS_EP_TIMEOUT = 2 };
/* Loads every kernel of the library on the current device now.  Under CUDA lazy loading a
 * kernel's first launch waits for the device to go idle, which never happens while a peer's
 * dymoe_ep_barrier spins waiting for this rank (the barrier then times out).
 * dymoe_ep_window_alloc calls it; call it yourself before the first barrier otherwise.
 * Errors: CUDA.                                                                               */
int dymoe_preload(void);
typedef struct dymoe_ep_window {
  int P, rank, M, Hd, cap_rows, parity;
  void* const* peers;
} dymoe_ep_window;
size_t dymoe_ep_window_bytes(int P, int M, int Hd, int cap_rows);
int dymoe_ep_window_alloc(size_t bytes, void** base, void* ipc_handle);
int dymoe_ep_window_open(const void* ipc_handle, void** base);
int dymoe_ep_window_close(void* base);
int dymoe_ep_window_free(void* base);
int dymoe_ep_publish_counts(const dymoe_ep_window* w, const int32_t* expert_off,
                            dymoe_stream_t stream);
int dymoe_ep_barrier(const dymoe_ep_window* w, uint32_t epoch, uint32_t* status,
                     dymoe_stream_t stream);
/* x [T][Hd] bf16; expert_off [M+1], perm_token [T*k] from dymoe_permute (skips dropped);
 * recv_off [M_loc+1] i32 out, M_loc = experts owned by this rank.  Rows that would exceed
 * cap_rows are not stored and set DYMOE_STATUS_EP_TIMEOUT's sibling bit
 * DYMOE_STATUS_EP_OVERFLOW in *status.                                                         */
enum { DYMOE_STATUS_EP_OVERFLOW = 4 };
int dymoe_ep_dispatch(const dymoe_ep_window* w, const uint16_t* x, int T,
                      const int32_t* expert_off, const int32_t* perm_token, int32_t* recv_off,
                      uint32_t* status, dymoe_stream_t stream);
/* inv_row [T][k], topk_w [T][k], expert_off [M+1] of this rank's dymoe_permute; y [T][Hd]
 * (out_dtype) out.  Same result as dymoe_combine on the unsharded layer.  A live slot whose row
 * lies past cap_rows (it was never stored by the dispatch) contributes nothing and sets
 * DYMOE_STATUS_EP_OVERFLOW in *status (nullable).                                             */
int dymoe_ep_combine(const dymoe_ep_window* w, const int32_t* inv_row, const float* topk_w,
                     int T, int k, const int32_t* expert_off, int renorm, int out_dtype, void* y,
                     uint32_t* status, dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* The whole layer, one step: route -> score -> assign -> permute -> FFN
 * -> combine, all on `stream` with no host synchronisation (graph-capturable).               */
typedef struct dymoe_fwd_opts {
  int phase;                 /* DYMOE_PREFILL (Eq. 1-2) or DYMOE_DECODE (Eq. 3) */
  int layer, num_layers;     /* l and L of Eq. 4 */
  dymoe_ladder ladder;
  const float* attn_mass;    /* prefill: [heads][T] f32 (R1) */
  int heads;
  int k_tokens;              /* prefill: 0 => ceil(0.2 T) */
  int ffn_mode;              /* -1 = choose (DECODE kernels when phase == DECODE), else as in
                                dymoe_expert_ffn */
  int out_dtype;             /* DYMOE_OUT_F32 (parity) or DYMOE_OUT_BF16 */
  const uint8_t* forced_bits;/* device [M], nullable: bypass score/assign (uniform sweeps) */
  void* prof_events[3];      /* nullable cudaEvent_t's recorded on `stream` before the gate/up
                                (W1/W3) FFN kernel, between it and the down (W2) kernel, and
                                after the down kernel (live per-kernel timing for benchmarks) */
  const uint16_t* residual;  /* device [T][Hd] bf16, nullable: the residual stream of a layer
                                stack (x_{l+1} = bf16(x_l + y_l)).  When set the
                                combine adds it after the slot sum (one fp32 add per element)
                                before the output rounding: y = out_dtype(residual + sum).  May
                                alias x but not y. */
} dymoe_fwd_opts;

/* Workspace: one device buffer of dymoe_workspace_size(...) bytes (256-byte aligned); it holds
 * every intermediate.  dymoe_workspace_views returns pointers into it (valid after the step
 * completes on the stream) for inspection: */
typedef struct dymoe_ws_views {
  int32_t* topk_idx;   /* [T][k] */
  float* topk_w;       /* [T][k] */
  float* probs;        /* [T][M] */
  float* importance;   /* [M] */
  int32_t* heavy;      /* [k_tokens] (prefill) */
  uint8_t* bits;       /* [M] */
  uint8_t* active;     /* [M] */
  int32_t* expert_off; /* [M+1] */
  int32_t* perm_token; /* [T*k] */
  int32_t* perm_slot;  /* [T*k] */
  int32_t* inv_row;    /* [T][k] */
  uint16_t* h;         /* [T*k][F] */
  float* y_perm;       /* [T*k][Hd] */
  uint32_t* status;    /* [1] */
  void* score_scratch;
} dymoe_ws_views;

size_t dymoe_workspace_size(const dymoe_layer* layer, int T);
int dymoe_workspace_views(const dymoe_layer* layer, int T, void* workspace,
                          dymoe_ws_views* views);

/* x [T][Hd] bf16, logits [T][M] f32, y [T][Hd] (out_dtype).  T = 0 is a no-op. */
int dymoe_moe_forward(const dymoe_layer* layer, const uint16_t* x, const float* logits, int T,
                      const dymoe_fwd_opts* opts, void* y, void* workspace, size_t ws_bytes,
                      dymoe_stream_t stream);

/* Synchronises `stream`, returns DYMOE_OK or DYMOE_ERR_DEVICE if a status bit is set in the
 * workspace's status word (*bits_out receives the word, nullable); clears the word.           */
int dymoe_check_status(const dymoe_layer* layer, int T, void* workspace, uint32_t* bits_out,
                       dymoe_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* The expert-parallel layer (BASELINE.json north_star "expert-parallel partitioning across 2, 4
 * and 8 GPUs"; PAPER.md P:203 steps ③-④ with the experts spread over P
 * GPUs).  Expert e lives on rank floor(e P / M) (contiguous blocks); each rank holds a
 * dymoe_layer of its own experts only (k_route = 1) and calls dymoe_moe_forward_ep with its own
 * tokens.  One step, every part inside the library:
 *   route + score the local tokens; make the importance GLOBAL (sum over ranks: exact counts in
 *   prefill, gate sums in decode; identical on every rank, so every rank assigns identical bits,
 *   Eq. 4-5); permute by expert (= by destination rank); send every routed row to its owner;
 *   the owner runs its experts' fused-dequant FFN on the rows it received (expert-major order:
 *   expert, source rank, source order); the rows come back and are combined with the routing
 *   weights (reading D12) -- the same result as dymoe_moe_forward on the unsharded layer.
 * Transports (dymoe_ep_config.transports, a mask; the call picks one):
 *   DYMOE_EP_NCCL  a communicator the handle owns (ncclCommInitRank on the caller's unique id;
 *                  libnccl.so.2 is loaded at dymoe_ep_create): importance all-reduce, count
 *                  all-gather, then grouped send/recv of exactly the rows each (source, expert)
 *                  pair exchanges -- straight into the expert-major receive rows and back into
 *                  the source's permuted order.  One host synchronisation per step (the count
 *                  matrix sizes the sends).
 *   DYMOE_EP_PEER  the symmetric windows above, mapped into every rank (dymoe_ep_connect): the
 *                  importance and per-expert counts go into every window, dispatch is the row
 *                  gather fused with the store into the owner's window, combine is the remote
 *                  load fused with the weighted combine; 3 device flag barriers, NO host
 *                  synchronisation (CUDA-graph capturable).  Needs peer access (NVLink /
 *                  NVSwitch) or one device.
 * Placements (the call's `placement`):
 *   DYMOE_EP_ALL_TO_ALL   every rank brings its own tokens (weak scaling), as above;
 *   DYMOE_EP_REPLICATED   decode with the SAME batch x on every rank (T <= 64): every rank
 *                  routes / scores / assigns the batch (identical, no exchange), runs its own
 *                  experts on the pairs routed to them, combines them with weights renormalised
 *                  over the global live set (D12), and the partial outputs are summed over the
 *                  ranks in rank order (NCCL all-reduce, or each rank's partial in its window
 *                  read by every rank after one barrier).
 * Requirements: every rank calls dymoe_moe_forward_ep the same number of times with the same
 * opts (phase, layer, ladder), placement and transport; T <= max_tokens; T_peer_max >= every
 * rank's T this step (0 = T); the ladder's m_mode may be ACTIVE (an expert is active if any rank
 * routes a token to it).  Device faults (barrier timeout, window overflow, a width not resident
 * on its owner) set bits of the step's status word (dymoe_ep_check_status).
 * Errors: INVALID (names the field), NCCL (communicator creation or a collective failed, message
 * has NCCL's error string; also when libnccl.so.2 cannot be loaded), CUDA, WORKSPACE.          */
typedef struct dymoe_ep dymoe_ep;
enum { DYMOE_EP_NCCL = 1, DYMOE_EP_PEER = 2 };
enum { DYMOE_EP_ALL_TO_ALL = 0, DYMOE_EP_REPLICATED = 1 };
#define DYMOE_EP_UID_BYTES 128
#define DYMOE_EP_IPC_BYTES 64
typedef struct dymoe_ep_config {
  int M, k_route, hidden, ffn;   /* the whole layer's shape (M experts over the ranks) */
  int max_tokens;                /* upper bound of T on any rank in any step */
  int transports;                /* DYMOE_EP_NCCL | DYMOE_EP_PEER */
} dymoe_ep_config;
/* An NCCL unique id (DYMOE_EP_UID_BYTES bytes, host) to broadcast from rank 0 to the others. */
int dymoe_ep_unique_id(void* uid);
/* Collective over the P ranks when nccl_uid != NULL (ncclCommInitRank on the current device).
 * Allocates this rank's window (cap = max_tokens * k_route * P rows).  With DYMOE_EP_PEER and a
 * communicator, the windows are exchanged over it (CUDA IPC handles all-gathered) and opened:
 * the handle is ready.  Without a communicator (nccl_uid = NULL, PEER only) the caller exchanges
 * the bases itself (dymoe_ep_window_base) and calls dymoe_ep_connect.                         */
int dymoe_ep_create(int rank, int world, const void* nccl_uid, const dymoe_ep_config* cfg,
                    dymoe_ep** out);
/* This rank's window base (device pointer) and its CUDA IPC handle (DYMOE_EP_IPC_BYTES, nullable). */
int dymoe_ep_window_base(const dymoe_ep* ep, void** base, void* ipc_handle);
/* peer_bases: host array [P] of every rank's window base valid in this process (the same
 * pointers for ranks that are threads of one process; dymoe_ep_window_open results otherwise). */
int dymoe_ep_connect(dymoe_ep* ep, void* const* peer_bases);
/* Workspace of one dymoe_moe_forward_ep call (device, 256-byte aligned). */
size_t dymoe_ep_workspace_size(const dymoe_ep* ep, int T, int T_peer_max, int placement);
/* Pointers into the workspace (as dymoe_workspace_views; `importance` is the global vector,
 * `expert_off` / `perm_*` / `inv_row` this rank's permutation, h / y_perm NULL). */
int dymoe_ep_workspace_views(const dymoe_ep* ep, int T, int T_peer_max, int placement,
                             void* workspace, dymoe_ws_views* views);
/* local: this rank's experts (dymoe_layer with M_loc = its block, k_route = 1, same hidden /
 * ffn).  x [T][Hd] bf16, logits [T][M] f32 device; y [T][Hd] (opts->out_dtype) out; opts as for
 * dymoe_moe_forward (forced_bits, prof_events and ffn_mode included; residual allowed).       */
int dymoe_moe_forward_ep(dymoe_ep* ep, const dymoe_layer* local, int transport, int placement,
                         const uint16_t* x, const float* logits, int T, int T_peer_max,
                         const dymoe_fwd_opts* opts, void* y, void* workspace, size_t ws_bytes,
                         dymoe_stream_t stream);
/* Host-side exchange plan of one all-to-all step -- exactly what the NCCL transport sends and
 * receives (exported so that the plan is checked without a GPU, tests/test_ep_gloo.py).
 *   counts [P][M] i32 host: rows rank src routes to expert e this step (after skips);
 *   send_off [M+1] i64 out: this rank's permuted rows of expert e are [send_off[e], send_off[e+1])
 *     and go to owner(e) as ONE message;
 *   recv_base [M_loc][P] i64 out: first receive row of (local expert el, source src): the rows
 *     are expert-major (local expert, then source rank, then the source's order);
 *   recv_off [M_loc+1] i32 out: local expert el's receive rows [recv_off[el], recv_off[el+1]).
 * Message order between a pair of ranks (NCCL matches sends and receives in order): the sender
 * walks the receiver's experts ascending, the receiver walks its own experts ascending; empty
 * messages are skipped on both sides.  The outputs return along the same chunks reversed.
 * Errors: INVALID (P, M, rank, negative counts, > 2^31 received rows).                        */
int dymoe_ep_plan_host(int P, int M, int rank, const int32_t* counts, int64_t* send_off,
                       int64_t* recv_base, int32_t* recv_off);
/* Synchronises `stream`; DYMOE_ERR_DEVICE if the step's status word (workspace) has a bit set
 * (*bits_out receives it, nullable); clears it. */
int dymoe_ep_check_status(const dymoe_ep* ep, int T, int T_peer_max, int placement,
                          void* workspace, uint32_t* bits_out, dymoe_stream_t stream);
int dymoe_ep_destroy(dymoe_ep* ep);

/* Last error message of the calling thread ("" if none). */
const char* dymoe_last_error(void);
/* Library version string. */
const char* dymoe_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DYMOE_H */
