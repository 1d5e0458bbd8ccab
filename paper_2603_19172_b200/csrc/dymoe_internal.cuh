// Internal declarations shared by the DyMoE sm_100a kernels and the C-ABI host layer.
// Nothing here is visible through include/dymoe.h.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <vector>

#include "../../include/dymoe.h"

namespace dymoe {
struct DevExpert;
}
struct dymoe_layer {
  int M, k, Hd, F;
  std::vector<dymoe::DevExpert> host;
  dymoe::DevExpert* dev = nullptr;
  uint32_t* meta_pool = nullptr;   // derived dequant metadata of every resident quantized matrix
  CUtensorMap* tmap_pool = nullptr;   // TMA descriptors of every resident matrix (device)
};

namespace dymoe {

// Kernel preloading.  Under CUDA lazy loading (the default) a kernel's first launch loads it, and
// loading waits for the device to go idle -- which never happens while a peer rank's
// dymoe_ep_barrier kernel spins waiting for this rank.  cudaFuncGetAttributes loads a kernel
// without launching it; each translation unit lists its kernels in a preload_* function.
template <class... K>
inline cudaError_t preload_kernels(K... k) {
  cudaError_t r = cudaSuccess;
  cudaFuncAttributes fa;
  ((r = (r == cudaSuccess ? cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(k)) : r)), ...);
  return r;
}
cudaError_t preload_route_score();
cudaError_t preload_permute_combine();
cudaError_t preload_ffn_decode();
cudaError_t preload_ffn_prefill();
cudaError_t preload_quantize();
cudaError_t preload_attn_mass();
cudaError_t preload_predict();
cudaError_t preload_norm();
cudaError_t preload_api();

// ------------------------------------------------------------------------------------------
// Device-side expert table (one entry per expert; copied to device by dymoe_layer_create).
struct DevQMat {
  const uint32_t* codes;
  const float* scales;
  const uint8_t* zeros;
  // Derived by the layer handle (dymoe_layer_create / refresh), owned by it: per group
  // (bf16 bits of RNE_bf16(scale)) << 16 | zero — exactly the two values dequant (D17) consumes,
  // in one 4-byte word — stored group-major, meta[g * N + n], so that the words of consecutive
  // rows for one group are contiguous (one TMA box per 16-row tile in the decode kernels,
  // coalesced per-row loads in the prefill producer).
  const uint32_t* meta;
  // TMA descriptors (device memory, owned by the layer handle): codes as a 2-D u8 tensor
  // {row bytes, N} with 128 x 16 boxes, 128-byte swizzle; meta as a u32 tensor {N, K / 128}
  // with 16 x (groups per 128-byte item) boxes -- 3-D {.., 2} for W1, covering the adjacent W1
  // and W3 meta with one box (W3's tm_meta is null); 2-D for W2.
  const CUtensorMap* tm_codes;
  const CUtensorMap* tm_meta;
  // prefill producer boxes: codes {64 k of 128 rows} (Int8 64-byte, Int4 32-byte swizzle, Int2
  // none) and the 128 rows' words of one group (meta {128, 1})
  const CUtensorMap* tm_raw;
  const CUtensorMap* tm_rawmeta;
};
// meta[g * N + n] = bf16bits(RNE(scales[n * gpr + g])) << 16 | zeros[n * gpr + g]
cudaError_t launch_build_meta(const float* scales, const uint8_t* zeros, int N, int gpr,
                              uint32_t* meta, cudaStream_t s);
struct DevExpert {
  const uint16_t* w[3];        // bf16 masters W1, W3, W2
  const CUtensorMap* tm_w[3];  // their TMA descriptors (u8 {2K, N}, 128 x 16 boxes, swizzled)
  const CUtensorMap* tm_wp[3]; // prefill B tiles: bf16 {K, N}, 64 x 128 boxes, 128-byte swizzle
  DevQMat q[3][3];             // [width idx: int8, int4, int2][matrix: W1, W3, W2]
};

__host__ __device__ inline int width_index(int bits) {
  return bits == 8 ? 0 : bits == 4 ? 1 : bits == 2 ? 2 : -1;
}

// Sets the thread-local error message returned by dymoe_last_error (dymoe_api.cu); returns code.
int set_error(int code, const char* fmt, ...);
void clear_error();

// ------------------------------------------------------------------------------------------
// Launchers (each returns cudaGetLastError() of its launch).
cudaError_t launch_route(const float* logits, int T, int M, int k, int32_t* topk_idx,
                         float* topk_w, float* probs, cudaStream_t s);

cudaError_t launch_score_prefill(const float* attn, int H, const int32_t* topk_idx, int T,
                                 int M, int k, int k_tokens, float* importance, int32_t* heavy,
                                 float* S_scratch, cudaStream_t s);
cudaError_t launch_score_decode(const float* logits, int B, int M, float* importance,
                                cudaStream_t s);

struct AssignParams {
  int M, k_route, n_tiers, clamp_to_k, m_active;
  int bits[DYMOE_MAX_TIERS];
  double r[DYMOE_MAX_TIERS - 1];   // host-evaluated Eq. 4 per threshold
};
// active_mask (nullable) or, when active_mask == nullptr and m_active, the mask is derived
// from topk_idx [T][k].  active_out (nullable) receives the derived mask.
cudaError_t launch_assign(const float* importance, const uint8_t* active_mask,
                          const int32_t* topk_idx, int T, const AssignParams& p, uint8_t* bits,
                          uint8_t* active_out, cudaStream_t s);

// Fused decode front (route -> [score -> assign] -> permute), one single-CTA launch; the same
// arithmetic as launch_route + launch_score_decode + launch_assign + launch_permute.
constexpr int kFrontDecodeMaxT = 256;
cudaError_t launch_front_decode(const float* logits, int T, int M, int k, const AssignParams& p,
                                const uint8_t* forced_bits, int32_t* topk_idx, float* topk_w,
                                float* probs, float* importance, uint8_t* bits, uint8_t* active,
                                int32_t* expert_off, int32_t* perm_token, int32_t* perm_slot,
                                int32_t* inv_row, int32_t* active_list, cudaStream_t s);

cudaError_t launch_quantize(const dymoe_quant_job* jobs_host, int n_jobs, cudaStream_t s);

// scratch (nullable, permute_scratch_bytes): with it, pair lists of more than
// kPermMultiMinChunks chunks of 1024 pairs take the multi-CTA path (same arrays, bit for bit).
constexpr int kPermMultiMinChunks = 4;
size_t permute_scratch_bytes(int T, int k, int M);
cudaError_t launch_permute(const int32_t* topk_idx, int T, int k, int M, const uint8_t* bits,
                           int32_t* expert_off, int32_t* perm_token, int32_t* perm_slot,
                           int32_t* inv_row, int32_t* active_list, cudaStream_t s,
                           int32_t* scratch = nullptr);

struct FfnArgs {
  const DevExpert* experts;
  int M, k, Hd, F;
  const uint16_t* x;           // [T][Hd]
  int T;
  const uint8_t* bits;         // [M]
  const int32_t* expert_off;   // [M+1]
  const int32_t* perm_token;   // [T*k]
  const int32_t* active_list;  // [M+1]: [0] = count, then expert ids
  uint16_t* h;                 // [T*k][F]
  float* y_perm;               // [T*k][Hd]   (prefill kernels)
  float* y_part;               // [SK][part_rows][Hd] (decode kernels: W2 K-slice partials;
                               // prefill: scratch for the expert-ordered token rows of GEMM 1)
  int part_rows;               // row capacity of one partial slice (>= T*k)
  uint32_t* status;
  int min_items;               // decode: min 128-byte items per warp per tile (set by the launcher)
};
// Number of K-slices (and slice length) the decode W2 kernel splits F into.
int decode_w2_slices(int F);
int decode_w2_slice_k(int F);
// y_perm[r][n] = sum_s y_part[s][r][n] (slice order), r < rows (and < *rows_dev when non-null)
cudaError_t launch_reduce_parts(const float* y_part, int n_parts, int part_rows, int rows, int Hd,
                                float* y_perm, cudaStream_t s, const int32_t* rows_dev = nullptr);
// y[r][:] = 0 for r < min(cap_rows, *rows_dev) (the routed rows of a capacity-sized buffer)
cudaError_t launch_zero_rows(float* y, int Hd, int cap_rows, const int32_t* rows_dev, cudaStream_t s);
// ev (nullable, 3 entries, each nullable): recorded before W13, between W13 and W2, after W2.
cudaError_t launch_ffn_decode(const FfnArgs& a, cudaStream_t s, void* const* ev = nullptr);
cudaError_t launch_ffn_prefill(const FfnArgs& a, cudaStream_t s, void* const* ev = nullptr);
// 2-D tiled TMA descriptor over a row-major [d1][d0] tensor (stride1 bytes between rows), box
// b0 x b1, CUtensorMapDataType dt, swizzle swz (host; false if the driver rejects it)
bool encode_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t d0,
                    uint64_t d1, uint64_t stride1, uint32_t b0, uint32_t b1,
                    CUtensorMapSwizzle swz);

// Inside a stream capture the record becomes a graph event-record node (cudaEventRecordExternal),
// so the events time the kernels when the graph is replayed.
inline void record_ev(void* const* ev, int i, cudaStream_t s) {
  if (ev == nullptr || ev[i] == nullptr) return;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(reinterpret_cast<cudaEvent_t>(ev[i]), s, cudaEventRecordExternal);
  else
    cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[i]), s);
}

cudaError_t launch_predict_next(int phase, const uint16_t* h, const uint16_t* wg, int T, int Hd,
                                int M, int k, int t, float* logits, int32_t* topk_idx,
                                float* topk_w, float* probs, float* value, int32_t* experts,
                                float* priority, int32_t* n_out, cudaStream_t s);
cudaError_t launch_attention_mass(const uint16_t* Q, const uint16_t* K, int H, int T, int d,
                                  float scale, float* m_scratch, float* l_scratch, float* a_out,
                                  cudaStream_t s);
cudaError_t launch_renorm_weights(const int32_t* topk_idx, const float* topk_w, const uint8_t* bits,
                                  int T, int k, int renorm, float* w_out, cudaStream_t s);
cudaError_t launch_ep_plan(const int32_t* expert_off, int M, int P, int32_t* send_counts,
                           int32_t* row_expert, cudaStream_t s);
cudaError_t launch_gather_rows(const uint16_t* x, int Hd, const int32_t* rows, int n,
                               uint16_t* out, cudaStream_t s);

// y_perm may hold n_parts partial slices [n_parts][part_rows][Hd]; they are summed in slice order
// before weighting (n_parts = 1, part_rows ignored for a plain y_perm).
// residual (nullable, [T][Hd] bf16): added after the slot sum, before the output rounding.
cudaError_t launch_combine(const float* y_perm, int n_parts, int part_rows, const int32_t* inv_row,
                           const float* topk_w, int T, int k, int Hd, int renorm, int out_dtype,
                           void* y, cudaStream_t s, const uint16_t* residual = nullptr);
// u[t] = bf16(x[t] / sqrt(mean(x[t]^2) + eps))  (stack RMSNorm, Hd multiple of 8)
cudaError_t launch_rmsnorm(const uint16_t* x, int T, int Hd, float eps, uint16_t* u, cudaStream_t s);
// logits[t][e] = h[t] . wg[e] (fp32, accumulation depth <= Hd/32 + 5) + bias[e] (nullable)
cudaError_t launch_gate_logits(const uint16_t* h, const uint16_t* wg, const float* bias, int T,
                               int Hd, int M, float* logits, cudaStream_t s);

// ------------------------------------------------------------------------------------------
// Expert-parallel windows (ep_p2p.cu; include/dymoe.h "Expert-parallel dispatch and combine over
// peer memory").  One symmetric window per rank, mapped into every rank:
//   flags  u32[P]            barrier counters
//   cnt    i32[2][P][M]      cnt[parity][src][e]: rows rank src routes to expert e
//   imp    f32[2][P][M]      imp[parity][src][e]: rank src's local importance (global Eq. 2 / 3)
//   red    f32[2][R][Hd]     replicated decode: this rank's partial output (R = kEpRedRows)
//   recv_x bf16[cap][Hd]     received rows, expert-major (local expert, source, source order)
//   y_out  f32[cap][Hd]      the local experts' outputs, row-aligned with recv_x
constexpr int kEpMaxP = 64;
constexpr int kEpRedRows = 64;
struct EpWinLayout {
  size_t flags, cnt, imp, red, recv_x, y_out, total;
};
__host__ __device__ inline size_t ep_align256(size_t v) { return (v + 255) & ~size_t(255); }
__host__ __device__ inline EpWinLayout ep_win_layout(int P, int M, int Hd, int cap) {
  EpWinLayout L;
  L.flags = 0;
  L.cnt = ep_align256((size_t)P * 4);
  L.imp = L.cnt + ep_align256((size_t)2 * P * M * 4);
  L.red = L.imp + ep_align256((size_t)2 * P * M * 4);
  L.recv_x = L.red + ep_align256((size_t)2 * kEpRedRows * Hd * 4);
  L.y_out = L.recv_x + ep_align256((size_t)cap * Hd * 2);
  L.total = L.y_out + ep_align256((size_t)cap * Hd * 4);
  return L;
}
struct EpWin {
  int P, rank, M, Hd, cap, parity;
  char* const* peers;      // device array [P] of window bases as mapped in this process
  const uint8_t* bits;     // device [M], nullable: counts of experts with bits == 0 read as 0
  EpWinLayout L;
};
__host__ __device__ inline int ep_owner_of(int e, int M, int P) { return (int)(((long long)e * P) / M); }
__host__ __device__ inline int ep_first_of_owner(int o, int M, int P) {
  return (int)(((long long)o * M + P - 1) / P);
}
// cnt[parity][rank][e] = off[e+1] - off[e] into every window (dymoe_ep_publish_counts)
cudaError_t launch_ep_publish(const EpWin& w, const int32_t* off, cudaStream_t s);
// imp[parity][rank][*] = importance, cnt[parity][rank][e] = #(t, slot) with topk_idx == e (before
// any skip: readers mask by bits) into every window
cudaError_t launch_ep_publish_pre(const EpWin& w, const float* importance, const int32_t* topk_idx,
                                  int T, int k, cudaStream_t s);
// importance[e] = sum_src imp[parity][src][e] (src order, fp32: identical on every rank);
// active[e] = (sum_src cnt[parity][src][e] > 0) (nullable)
cudaError_t launch_ep_reduce_imp(const EpWin& w, float* importance, uint8_t* active, cudaStream_t s);
cudaError_t launch_ep_barrier(const EpWin& w, uint32_t epoch, uint32_t* status, cudaStream_t s);
cudaError_t launch_ep_dispatch(const EpWin& w, const uint16_t* x, const int32_t* off,
                               const int32_t* perm_token, int32_t* recv_off, uint32_t* status,
                               cudaStream_t s);
cudaError_t launch_ep_combine(const EpWin& w, const int32_t* inv_row, const float* topk_w, int T,
                              int k, const int32_t* off, int renorm, int out_dtype, void* y,
                              const uint16_t* residual, uint32_t* status, cudaStream_t s);
// y[t] = out_dtype(residual[t] + sum_src red[parity][t] of window src), src order, t < B
cudaError_t launch_ep_reduce_red(const EpWin& w, int B, int out_dtype, void* y,
                                 const uint16_t* residual, cudaStream_t s);
cudaError_t preload_ep();
cudaError_t preload_ep_layer();
// The expert FFN on expert-ordered rows whose count is on the device (expert_off[M] of `L`);
// cap_rows bounds it.  ws: dymoe_expert_ffn's scratch for cap_rows rows (dymoe_api.cu).
size_t ffn_ws_parts_bytes(const dymoe_layer* L, int rows);
int expert_ffn_rows(const dymoe_layer* L, int mode, const uint16_t* x, int cap_rows,
                    const uint8_t* bits, const int32_t* expert_off, const int32_t* perm_token,
                    uint16_t* h_ws, float* y_perm, uint32_t* status, void* ws, cudaStream_t s,
                    void* const* ev);
int assign_params(const dymoe_ladder* ladder, int M, int k_route, int layer, int num_layers,
                  AssignParams& p);

// ------------------------------------------------------------------------------------------
// Small device helpers.
__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

}  // namespace dymoe
