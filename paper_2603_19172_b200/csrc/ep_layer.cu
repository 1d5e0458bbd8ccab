// The expert-parallel layer behind the C ABI (include/dymoe.h "The expert-parallel layer";
// BASELINE.json north_star).  Host orchestration of one step on the
// caller's stream; every step of the math runs in libdymoe kernels, the bytes move either
// through a communicator the handle owns (NCCL, loaded at run time) or through the symmetric
// peer-memory windows of ep_p2p.cu (NVLink / NVSwitch loads and stores, device flag barriers).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <type_traits>
#include <vector>

#include "dymoe_internal.cuh"

using namespace dymoe;

namespace {

// ------------------------------------------------------------------------------------------
// NCCL, resolved from libnccl.so.2 at run time (the process's already-loaded copy if any, e.g.
// PyTorch's), so that the library itself loads on machines without NCCL.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
  char why[256] = {0};
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      snprintf(a.why, sizeof(a.why), "libnccl.so.2 not loadable: %s", dlerror());
      return a;
    }
    bool ok = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (fn == nullptr) {
        ok = false;
        snprintf(a.why, sizeof(a.why), "libnccl.so.2 lacks %s", name);
      }
    };
    get(a.GetUniqueId, "ncclGetUniqueId");
    get(a.CommInitRank, "ncclCommInitRank");
    get(a.CommDestroy, "ncclCommDestroy");
    get(a.AllReduce, "ncclAllReduce");
    get(a.AllGather, "ncclAllGather");
    get(a.Send, "ncclSend");
    get(a.Recv, "ncclRecv");
    get(a.GroupStart, "ncclGroupStart");
    get(a.GroupEnd, "ncclGroupEnd");
    get(a.GetErrorString, "ncclGetErrorString");
    a.ok = ok;
    return a;
  }();
  return api;
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return set_error(code, "%s", buf);
}

#define EP_ARG(cond, ...)                                    \
  do {                                                       \
    if (!(cond)) return fail(DYMOE_ERR_INVALID, __VA_ARGS__); \
  } while (0)
#define EP_CUDA(expr, where)                                                            \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) return fail(DYMOE_ERR_CUDA, "%s: %s", where, cudaGetErrorString(_e)); \
  } while (0)
#define EP_NCCL(expr, where)                                                               \
  do {                                                                                     \
    ncclResult_t _r = (expr);                                                              \
    if (_r != ncclSuccess)                                                                 \
      return fail(DYMOE_ERR_NCCL, "%s: %s", where, nccl().GetErrorString(_r));             \
  } while (0)

size_t al(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

struct dymoe_ep {
  int rank = 0, P = 1, M = 0, k = 0, Hd = 0, F = 0, max_T = 0, cap = 0, transports = 0;
  int first = 0, last = 0;   // owned experts [first, last)
  ncclComm_t comm = nullptr;
  char* win = nullptr;       // this rank's window
  size_t win_bytes = 0;
  std::vector<void*> opened;  // peers' windows opened through CUDA IPC (closed at destroy)
  char** peers_dev = nullptr; // [P] window bases as mapped here
  char** self_dev = nullptr;  // [1] own window (single-source reduction of an NCCL all-reduce)
  bool connected = false;
  uint32_t epoch = 0;
  int parity = 0;
  int32_t* host_cnt = nullptr;  // pinned [P][M] count matrix (NCCL path)
  int32_t* host_roff = nullptr; // pinned [M_loc + 1] receive offsets (NCCL path)
  int32_t* ident = nullptr;     // device [cap]: identity row map (the FFN reads received rows in place)
};

namespace {

struct EpWs {
  size_t topk_idx, topk_w, probs, imp_local, imp, heavy, bits, active, active_list, off,
      perm_token, perm_slot, inv_row, score_scratch, perm_scratch, status, cnt_local, cnt_all,
      x_send, y_back, recv_off, ffn_ws, h, idx_loc, bits_loc, wn, off_l, pt_l, ps_l, inv_l, total;
  int rows_cap;
};

size_t ffn_parts(int F, int Hd, int rows) {
  const size_t dec = (size_t)decode_w2_slices(F) * rows * Hd * sizeof(float);
  const size_t pre = (size_t)rows * Hd * 2;
  return dec > pre ? dec : pre;
}

EpWs ep_ws(const dymoe_ep* ep, int T, int Tp, int placement) {
  EpWs W{};
  size_t o = 0;
  auto take = [&](size_t b) {
    const size_t at = o;
    o = al(o + (b > 0 ? b : 1));
    return at;
  };
  const int M = ep->M, k = ep->k, Hd = ep->Hd;
  const size_t TK = (size_t)(T > 0 ? T : 1) * k;
  W.rows_cap = placement == DYMOE_EP_REPLICATED
                   ? (int)TK
                   : (int)std::min<long long>(ep->cap, (long long)(Tp > T ? Tp : T) * k * ep->P);
  if (W.rows_cap < 1) W.rows_cap = 1;
  const size_t R = (size_t)W.rows_cap;
  W.topk_idx = take(TK * 4);
  W.topk_w = take(TK * 4);
  W.probs = take((size_t)(T > 0 ? T : 1) * M * 4);
  W.imp_local = take((size_t)M * 4);
  W.imp = take((size_t)M * 4);
  W.heavy = take((size_t)(T > 0 ? T : 1) * 4);
  W.bits = take((size_t)M + 1);
  W.active = take((size_t)M);
  W.active_list = take((size_t)3 * (M + 2) * 4);
  W.off = take((size_t)(M + 2) * 4);
  W.perm_token = take(TK * 4);
  W.perm_slot = take(TK * 4);
  W.inv_row = take(TK * 4);
  W.score_scratch = take((size_t)(T > 0 ? T : 1) * 4);
  W.perm_scratch = take(permute_scratch_bytes(T, k, M + 1));
  W.status = take(4);
  W.cnt_local = take((size_t)M * 4);
  W.cnt_all = take((size_t)ep->P * M * 4);
  const bool nccl_a2a = placement == DYMOE_EP_ALL_TO_ALL && (ep->transports & DYMOE_EP_NCCL);
  W.x_send = take(nccl_a2a ? TK * Hd * 2 : 0);
  W.y_back = take(nccl_a2a || placement == DYMOE_EP_REPLICATED ? TK * Hd * 4 : 0);
  W.recv_off = take((size_t)(M + 1) * 4);
  W.ffn_ws = take(al((size_t)3 * (M + 2) * 4) + al(ffn_parts(ep->F, Hd, (int)R)));
  W.h = take(R * ep->F * 2);
  const bool rep = placement == DYMOE_EP_REPLICATED;
  W.idx_loc = take(rep ? TK * 4 : 0);
  W.bits_loc = take(rep ? (size_t)M + 1 : 0);
  W.wn = take(rep ? TK * 4 : 0);
  W.off_l = take(rep ? (size_t)(M + 2) * 4 : 0);
  W.pt_l = take(rep ? TK * 4 : 0);
  W.ps_l = take(rep ? TK * 4 : 0);
  W.inv_l = take(rep ? TK * 4 : 0);
  W.total = o;
  return W;
}

template <class T_>
T_* at(void* ws, size_t off) {
  return reinterpret_cast<T_*>(reinterpret_cast<char*>(ws) + off);
}

EpWin win_of(const dymoe_ep* ep, const uint8_t* bits) {
  EpWin w{};
  w.P = ep->P;
  w.rank = ep->rank;
  w.M = ep->M;
  w.Hd = ep->Hd;
  w.cap = ep->cap;
  w.parity = ep->parity;
  w.peers = ep->peers_dev;
  w.bits = bits;
  w.L = ep_win_layout(ep->P, ep->M, ep->Hd, ep->cap);
  return w;
}

// per-expert counts of this rank's permutation (post-skip): cnt[e] = off[e+1] - off[e]
__global__ void k_counts_from_off(const int32_t* __restrict__ off, int M, int32_t* __restrict__ cnt) {
  for (int e = threadIdx.x; e < M; e += blockDim.x) cnt[e] = off[e + 1] - off[e];
}
// histogram of the routing (pre-skip)
__global__ void k_route_hist(const int32_t* __restrict__ idx, int n, int M, int32_t* __restrict__ h) {
  __shared__ int c[DYMOE_MAX_EXPERTS];
  for (int e = threadIdx.x; e < M; e += blockDim.x) c[e] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&c[idx[i]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < M; e += blockDim.x) h[e] = c[e];
}
__global__ void k_active_from_counts(const int32_t* __restrict__ cnt, int M, uint8_t* __restrict__ a) {
  for (int e = threadIdx.x; e < M; e += blockDim.x) a[e] = cnt[e] > 0;
}
// replicated decode: the local view of the routing -- this rank's experts keep their index
// (shifted by `first`) and width, every other expert maps to one extra skipped slot M_loc
__global__ void k_local_view(const int32_t* __restrict__ idx, int n, int first, int last,
                             const uint8_t* __restrict__ bits, int32_t* __restrict__ idx_loc,
                             uint8_t* __restrict__ bits_loc) {
  const int M_loc = last - first;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e = idx[i];
    idx_loc[i] = (e >= first && e < last) ? e - first : M_loc;
  }
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= M_loc; e += blockDim.x) bits_loc[e] = e < M_loc ? bits[first + e] : 0;
}
__global__ void k_iota(int32_t* __restrict__ v, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

int check_cfg(const dymoe_ep_config* c, int rank, int world) {
  EP_ARG(c != nullptr, "cfg: must not be NULL");
  EP_ARG(c->M >= 1 && c->M <= DYMOE_MAX_EXPERTS, "cfg.M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  EP_ARG(c->k_route >= 1 && c->k_route <= c->M && c->k_route <= 8,
         "cfg.k_route: must satisfy 1 <= k_route <= min(M, 8)");
  EP_ARG(c->hidden > 0 && c->hidden % 128 == 0, "cfg.hidden: must be a positive multiple of 128");
  EP_ARG(c->ffn > 0 && c->ffn % 128 == 0, "cfg.ffn: must be a positive multiple of 128");
  EP_ARG(c->max_tokens >= 1, "cfg.max_tokens: must be >= 1");
  EP_ARG(c->transports >= 1 && c->transports <= (DYMOE_EP_NCCL | DYMOE_EP_PEER),
         "cfg.transports: must be a non-empty mask of DYMOE_EP_NCCL | DYMOE_EP_PEER");
  EP_ARG(world >= 1 && world <= c->M && world <= kEpMaxP, "world: must satisfy 1 <= world <= min(M, %d)",
         kEpMaxP);
  EP_ARG(rank >= 0 && rank < world, "rank: must be in [0, world)");
  EP_ARG((long long)c->max_tokens * c->k_route * world < (1ll << 31), "cfg.max_tokens: too large");
  return DYMOE_OK;
}

void destroy(dymoe_ep* ep) {
  if (ep == nullptr) return;
  cudaDeviceSynchronize();
  for (void* b : ep->opened) cudaIpcCloseMemHandle(b);
  if (ep->comm != nullptr && nccl().ok) nccl().CommDestroy(ep->comm);
  if (ep->win) cudaFree(ep->win);
  if (ep->peers_dev) cudaFree(ep->peers_dev);
  if (ep->self_dev) cudaFree(ep->self_dev);
  if (ep->ident) cudaFree(ep->ident);
  if (ep->host_cnt) cudaFreeHost(ep->host_cnt);
  if (ep->host_roff) cudaFreeHost(ep->host_roff);
  delete ep;
}

int do_connect(dymoe_ep* ep, void* const* bases) {
  std::vector<char*> b(ep->P);
  for (int p = 0; p < ep->P; ++p) {
    EP_ARG(bases[p] != nullptr, "peer_bases[%d]: must not be NULL", p);
    b[p] = reinterpret_cast<char*>(bases[p]);
  }
  EP_ARG(b[ep->rank] == ep->win, "peer_bases[rank]: must be this rank's own window");
  EP_CUDA(cudaMemcpy(ep->peers_dev, b.data(), sizeof(char*) * ep->P, cudaMemcpyHostToDevice),
          "dymoe_ep_connect");
  ep->connected = true;
  return DYMOE_OK;
}

// ------------------------------------------------------------------------------------------
// The steps.  Every function returns DYMOE_OK or an error (set_error) and only enqueues work on s.

// local importance (Eq. 2 counts of this rank's heavy hitters / Eq. 3 gate sums of its tokens)
int local_importance(const dymoe_ep* ep, const dymoe_fwd_opts* o, int T, int k_tokens,
                     const float* logits, void* ws, const EpWs& W, cudaStream_t s) {
  const int M = ep->M;
  float* imp = at<float>(ws, W.imp_local);
  if (T == 0) {
    EP_CUDA(cudaMemsetAsync(imp, 0, (size_t)M * 4, s), "importance");
    return DYMOE_OK;
  }
  if (o->phase == DYMOE_PREFILL) {
    EP_CUDA(launch_score_prefill(o->attn_mass, o->heads, at<int32_t>(ws, W.topk_idx), T, M, ep->k,
                                 k_tokens, imp, at<int32_t>(ws, W.heavy),
                                 at<float>(ws, W.score_scratch), s),
            "score");
  } else if (T == 1 && ep->P > 1) {
    // one token: its gate row g (Eq. 3; the logit row of the unsharded B = 1 ranking is not
    // additive over ranks)
    EP_CUDA(cudaMemcpyAsync(imp, at<float>(ws, W.probs), (size_t)M * 4, cudaMemcpyDeviceToDevice, s),
            "importance");
  } else {
    EP_CUDA(launch_score_decode(logits, T, M, imp, s), "score");
  }
  return DYMOE_OK;
}

int a2a_peer(dymoe_ep* ep, const dymoe_layer* local, const dymoe_fwd_opts* o, const AssignParams& ap,
             const uint16_t* x, const float* logits, int T, void* y, void* ws, const EpWs& W,
             int k_tokens, cudaStream_t s) {
  const int M = ep->M, k = ep->k;
  uint32_t* status = at<uint32_t>(ws, W.status);
  uint8_t* bits = at<uint8_t>(ws, W.bits);
  const uint8_t* use_bits = o->forced_bits ? o->forced_bits : bits;
  EpWin w0 = win_of(ep, nullptr);
  int rc = local_importance(ep, o, T, k_tokens, logits, ws, W, s);
  if (rc) return rc;
  EP_CUDA(launch_ep_publish_pre(w0, at<float>(ws, W.imp_local), at<int32_t>(ws, W.topk_idx), T, k, s),
          "publish");
  EP_CUDA(launch_ep_barrier(w0, ++ep->epoch, status, s), "barrier");
  EP_CUDA(launch_ep_reduce_imp(w0, at<float>(ws, W.imp), at<uint8_t>(ws, W.active), s), "reduce");
  if (o->forced_bits == nullptr)
    EP_CUDA(launch_assign(at<float>(ws, W.imp), at<uint8_t>(ws, W.active), nullptr, 0, ap, bits,
                          nullptr, s),
            "assign");
  EP_CUDA(launch_permute(at<int32_t>(ws, W.topk_idx), T, k, M, use_bits, at<int32_t>(ws, W.off),
                         at<int32_t>(ws, W.perm_token), at<int32_t>(ws, W.perm_slot),
                         at<int32_t>(ws, W.inv_row), at<int32_t>(ws, W.active_list), s,
                         at<int32_t>(ws, W.perm_scratch)),
          "permute");
  const EpWin w = win_of(ep, use_bits);
  int32_t* recv_off = at<int32_t>(ws, W.recv_off);
  EP_CUDA(launch_ep_dispatch(w, x, at<int32_t>(ws, W.off), at<int32_t>(ws, W.perm_token), recv_off,
                             status, s),
          "dispatch");
  EP_CUDA(launch_ep_barrier(w, ++ep->epoch, status, s), "barrier");
  const int M_loc = ep->last - ep->first;
  if (M_loc > 0) {
    const int mode = o->ffn_mode == -1 ? o->phase : o->ffn_mode;
    rc = expert_ffn_rows(local, mode, reinterpret_cast<const uint16_t*>(ep->win + w.L.recv_x),
                         W.rows_cap, use_bits + ep->first, recv_off, ep->ident,
                         at<uint16_t>(ws, W.h), reinterpret_cast<float*>(ep->win + w.L.y_out),
                         status, at<void>(ws, W.ffn_ws), s, o->prof_events);
    if (rc) return rc;
  }
  EP_CUDA(launch_ep_barrier(w, ++ep->epoch, status, s), "barrier");
  EP_CUDA(launch_ep_combine(w, at<int32_t>(ws, W.inv_row), at<float>(ws, W.topk_w), T, k,
                            at<int32_t>(ws, W.off), o->ladder.renorm_on_skip, o->out_dtype, y,
                            o->residual, status, s),
          "combine");
  ep->parity ^= 1;
  return DYMOE_OK;
}

int a2a_nccl(dymoe_ep* ep, const dymoe_layer* local, const dymoe_fwd_opts* o, const AssignParams& ap,
             const uint16_t* x, const float* logits, int T, void* y, void* ws, const EpWs& W,
             int k_tokens, cudaStream_t s) {
  const NcclApi& N = nccl();
  const int M = ep->M, k = ep->k, P = ep->P, Hd = ep->Hd;
  uint32_t* status = at<uint32_t>(ws, W.status);
  uint8_t* bits = at<uint8_t>(ws, W.bits);
  const uint8_t* use_bits = o->forced_bits ? o->forced_bits : bits;
  int rc = local_importance(ep, o, T, k_tokens, logits, ws, W, s);
  if (rc) return rc;
  // global importance (and, for ACTIVE mode, the global routing histogram)
  const bool act = ap.m_active != 0;
  if (act) {
    k_route_hist<<<1, 1024, 0, s>>>(at<int32_t>(ws, W.topk_idx), T * k, M, at<int32_t>(ws, W.cnt_local));
    EP_CUDA(cudaGetLastError(), "hist");
  }
  EP_NCCL(N.GroupStart(), "ncclGroupStart");
  EP_NCCL(N.AllReduce(at<float>(ws, W.imp_local), at<float>(ws, W.imp), M, ncclFloat32, ncclSum,
                      ep->comm, s),
          "ncclAllReduce(importance)");
  if (act)
    EP_NCCL(N.AllReduce(at<int32_t>(ws, W.cnt_local), at<int32_t>(ws, W.cnt_all), M, ncclInt32,
                        ncclSum, ep->comm, s),
            "ncclAllReduce(routing histogram)");
  EP_NCCL(N.GroupEnd(), "ncclGroupEnd");
  if (act) {
    k_active_from_counts<<<1, 256, 0, s>>>(at<int32_t>(ws, W.cnt_all), M, at<uint8_t>(ws, W.active));
    EP_CUDA(cudaGetLastError(), "active");
  }
  if (o->forced_bits == nullptr)
    EP_CUDA(launch_assign(at<float>(ws, W.imp), act ? at<uint8_t>(ws, W.active) : nullptr, nullptr,
                          0, ap, bits, nullptr, s),
            "assign");
  int32_t* off = at<int32_t>(ws, W.off);
  EP_CUDA(launch_permute(at<int32_t>(ws, W.topk_idx), T, k, M, use_bits, off,
                         at<int32_t>(ws, W.perm_token), at<int32_t>(ws, W.perm_slot),
                         at<int32_t>(ws, W.inv_row), at<int32_t>(ws, W.active_list), s,
                         at<int32_t>(ws, W.perm_scratch)),
          "permute");
  // the count matrix [P][M] on every rank: the one host synchronisation of the step
  k_counts_from_off<<<1, 256, 0, s>>>(off, M, at<int32_t>(ws, W.cnt_local));
  EP_CUDA(cudaGetLastError(), "counts");
  EP_NCCL(N.AllGather(at<int32_t>(ws, W.cnt_local), at<int32_t>(ws, W.cnt_all), M, ncclInt32,
                      ep->comm, s),
          "ncclAllGather(counts)");
  EP_CUDA(cudaMemcpyAsync(ep->host_cnt, at<int32_t>(ws, W.cnt_all), (size_t)P * M * 4,
                          cudaMemcpyDeviceToHost, s),
          "counts");
  EP_CUDA(cudaStreamSynchronize(s), "counts");
  const int32_t* C = ep->host_cnt;   // C[src][e]
  const int M_loc = ep->last - ep->first;
  std::vector<int64_t> soff(M + 1), rbase((size_t)M_loc * P + 1);
  rc = dymoe_ep_plan_host(P, M, ep->rank, C, soff.data(), rbase.data(), ep->host_roff);
  if (rc) return rc;
  const long long n_recv = ep->host_roff[M_loc];
  if (n_recv > ep->cap) return fail(DYMOE_ERR_INVALID, "T_peer_max/cfg.max_tokens: %lld rows received > window capacity %d", n_recv, ep->cap);
  const EpWin w = win_of(ep, use_bits);
  uint16_t* recv_x = reinterpret_cast<uint16_t*>(ep->win + w.L.recv_x);
  float* y_out = reinterpret_cast<float*>(ep->win + w.L.y_out);
  uint16_t* x_send = at<uint16_t>(ws, W.x_send);
  float* y_back = at<float>(ws, W.y_back);
  const int64_t R = soff[M];
  if (R > 0) EP_CUDA(launch_gather_rows(x, Hd, at<int32_t>(ws, W.perm_token), (int)R, x_send, s), "gather");
  // dispatch: one (expert, peer) chunk per message, straight to its expert-major rows
  EP_NCCL(N.GroupStart(), "ncclGroupStart");
  for (int d = 0; d < P; ++d) {
    const int f = ep_first_of_owner(d, M, P), l = ep_first_of_owner(d + 1, M, P);
    for (int e = f; e < l; ++e) {
      const int64_t c = soff[e + 1] - soff[e];
      if (c > 0)
        EP_NCCL(N.Send(x_send + soff[e] * Hd, (size_t)c * Hd, ncclBfloat16, d, ep->comm, s), "ncclSend(rows)");
    }
  }
  for (int src = 0; src < P; ++src)
    for (int el = 0; el < M_loc; ++el) {
      const int64_t c = C[(size_t)src * M + ep->first + el];
      if (c > 0)
        EP_NCCL(N.Recv(recv_x + rbase[(size_t)el * P + src] * Hd, (size_t)c * Hd, ncclBfloat16, src,
                       ep->comm, s),
                "ncclRecv(rows)");
    }
  EP_NCCL(N.GroupEnd(), "ncclGroupEnd");
  int32_t* recv_off = at<int32_t>(ws, W.recv_off);
  EP_CUDA(cudaMemcpyAsync(recv_off, ep->host_roff, (size_t)(M_loc + 1) * 4, cudaMemcpyHostToDevice, s),
          "recv offsets");
  if (M_loc > 0 && n_recv > 0) {
    const int mode = o->ffn_mode == -1 ? o->phase : o->ffn_mode;
    rc = expert_ffn_rows(local, mode, recv_x, (int)n_recv, use_bits + ep->first, recv_off,
                         ep->ident, at<uint16_t>(ws, W.h), y_out, status, at<void>(ws, W.ffn_ws), s,
                         o->prof_events);
    if (rc) return rc;
  }
  // combine: the outputs go back chunk by chunk into the source's permuted order
  EP_NCCL(N.GroupStart(), "ncclGroupStart");
  for (int src = 0; src < P; ++src)
    for (int el = 0; el < M_loc; ++el) {
      const int64_t c = C[(size_t)src * M + ep->first + el];
      if (c > 0)
        EP_NCCL(N.Send(y_out + rbase[(size_t)el * P + src] * Hd, (size_t)c * Hd, ncclFloat32, src,
                       ep->comm, s),
                "ncclSend(outputs)");
    }
  for (int d = 0; d < P; ++d) {
    const int f = ep_first_of_owner(d, M, P), l = ep_first_of_owner(d + 1, M, P);
    for (int e = f; e < l; ++e) {
      const int64_t c = soff[e + 1] - soff[e];
      if (c > 0)
        EP_NCCL(N.Recv(y_back + soff[e] * Hd, (size_t)c * Hd, ncclFloat32, d, ep->comm, s), "ncclRecv(outputs)");
    }
  }
  EP_NCCL(N.GroupEnd(), "ncclGroupEnd");
  if (T > 0)
    EP_CUDA(launch_combine(y_back, 1, T * k, at<int32_t>(ws, W.inv_row), at<float>(ws, W.topk_w), T,
                           k, Hd, o->ladder.renorm_on_skip, o->out_dtype, y, s, o->residual),
            "combine");
  return DYMOE_OK;
}

int replicated(dymoe_ep* ep, const dymoe_layer* local, int transport, const dymoe_fwd_opts* o,
               const AssignParams& ap, const uint16_t* x, const float* logits, int T, void* y,
               void* ws, const EpWs& W, cudaStream_t s) {
  const int M = ep->M, k = ep->k, Hd = ep->Hd;
  uint32_t* status = at<uint32_t>(ws, W.status);
  uint8_t* bits = at<uint8_t>(ws, W.bits);
  const uint8_t* use_bits = o->forced_bits ? o->forced_bits : bits;
  // the whole batch, identical on every rank: score (Eq. 3 on the batch) and assign
  if (o->forced_bits == nullptr) {
    EP_CUDA(launch_score_decode(logits, T, M, at<float>(ws, W.imp), s), "score");
    EP_CUDA(launch_assign(at<float>(ws, W.imp), nullptr, at<int32_t>(ws, W.topk_idx), T, ap, bits,
                          at<uint8_t>(ws, W.active), s),
            "assign");
  }
  // combine weights against the global live set, then the local view of the routing
  float* wn = at<float>(ws, W.wn);
  EP_CUDA(launch_renorm_weights(at<int32_t>(ws, W.topk_idx), at<float>(ws, W.topk_w), use_bits, T, k,
                                o->ladder.renorm_on_skip, wn, s),
          "renorm");
  const int M_loc = ep->last - ep->first;
  int32_t* idx_loc = at<int32_t>(ws, W.idx_loc);
  uint8_t* bits_loc = at<uint8_t>(ws, W.bits_loc);
  k_local_view<<<1, 256, 0, s>>>(at<int32_t>(ws, W.topk_idx), T * k, ep->first, ep->last, use_bits,
                                 idx_loc, bits_loc);
  EP_CUDA(cudaGetLastError(), "local view");
  int32_t* off_l = at<int32_t>(ws, W.off_l);
  EP_CUDA(launch_permute(idx_loc, T, k, M_loc + 1, bits_loc, off_l, at<int32_t>(ws, W.pt_l),
                         at<int32_t>(ws, W.ps_l), at<int32_t>(ws, W.inv_l),
                         at<int32_t>(ws, W.active_list), s, at<int32_t>(ws, W.perm_scratch)),
          "permute");
  // local experts on their pairs (rows read from x through the permutation; the slot M_loc is
  // skipped, so off_l[M_loc] counts exactly the local rows)
  float* y_loc = at<float>(ws, W.y_back);
  if (M_loc > 0) {
    const int mode = o->ffn_mode == -1 ? DYMOE_DECODE : o->ffn_mode;
    int rc = expert_ffn_rows(local, mode, x, W.rows_cap, bits_loc, off_l, at<int32_t>(ws, W.pt_l),
                             at<uint16_t>(ws, W.h), y_loc, status, at<void>(ws, W.ffn_ws), s,
                             o->prof_events);
    if (rc) return rc;
  }
  // this rank's partial output (weights already renormalised globally: renorm = 0) into its
  // window's reduction slot, then the sum over the ranks in rank order
  const EpWin w = win_of(ep, use_bits);
  float* red_own = reinterpret_cast<float*>(ep->win + w.L.red) + (size_t)ep->parity * kEpRedRows * Hd;
  EP_CUDA(launch_combine(y_loc, 1, T * k, at<int32_t>(ws, W.inv_l), wn, T, k, Hd, 0, DYMOE_OUT_F32,
                         red_own, s),
          "partial combine");
  if (transport == DYMOE_EP_PEER) {
    EP_CUDA(launch_ep_barrier(w, ++ep->epoch, status, s), "barrier");
    EP_CUDA(launch_ep_reduce_red(w, T, o->out_dtype, y, o->residual, s), "reduce");
  } else {
    EP_NCCL(nccl().AllReduce(red_own, red_own, (size_t)T * Hd, ncclFloat32, ncclSum, ep->comm, s),
            "ncclAllReduce(outputs)");
    EpWin one = w;
    one.P = 1;
    one.rank = 0;
    one.peers = ep->self_dev;
    EP_CUDA(launch_ep_reduce_red(one, T, o->out_dtype, y, o->residual, s), "output");
  }
  ep->parity ^= 1;
  return DYMOE_OK;
}

}  // namespace

extern "C" {

int dymoe_ep_plan_host(int P, int M, int rank, const int32_t* counts, int64_t* send_off,
                       int64_t* recv_base, int32_t* recv_off) {
  EP_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  EP_ARG(P >= 1 && P <= M && P <= kEpMaxP, "P: must satisfy 1 <= P <= min(M, %d)", kEpMaxP);
  EP_ARG(rank >= 0 && rank < P, "rank: must be in [0, P)");
  EP_ARG(counts && send_off && recv_base && recv_off, "counts/send_off/recv_base/recv_off: must not be NULL");
  for (int i = 0; i < P * M; ++i) EP_ARG(counts[i] >= 0, "counts[%d]: must be >= 0", i);
  // this rank's rows in permuted (expert) order: expert e's rows start at send_off[e]
  send_off[0] = 0;
  for (int e = 0; e < M; ++e) send_off[e + 1] = send_off[e] + counts[(size_t)rank * M + e];
  // receive rows, expert-major: local expert, then source rank, then the source's order
  const int first = ep_first_of_owner(rank, M, P), M_loc = ep_first_of_owner(rank + 1, M, P) - first;
  int64_t n = 0;
  for (int el = 0; el < M_loc; ++el) {
    EP_ARG(n < (1ll << 31), "counts: more than 2^31 received rows");
    recv_off[el] = (int32_t)n;
    for (int src = 0; src < P; ++src) {
      recv_base[(size_t)el * P + src] = n;
      n += counts[(size_t)src * M + first + el];
    }
  }
  EP_ARG(n < (1ll << 31), "counts: more than 2^31 received rows");
  recv_off[M_loc] = (int32_t)n;
  clear_error();
  return DYMOE_OK;
}

int dymoe_ep_unique_id(void* uid) {
  EP_ARG(uid != nullptr, "uid: must not be NULL");
  const NcclApi& N = nccl();
  if (!N.ok) return fail(DYMOE_ERR_NCCL, "%s", N.why);
  ncclUniqueId id;
  EP_NCCL(N.GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == DYMOE_EP_UID_BYTES, "NCCL unique id size");
  memcpy(uid, &id, sizeof(id));
  clear_error();
  return DYMOE_OK;
}

int dymoe_ep_create(int rank, int world, const void* nccl_uid, const dymoe_ep_config* cfg,
                    dymoe_ep** out) {
  EP_ARG(out != nullptr, "out: must not be NULL");
  *out = nullptr;
  int rc = check_cfg(cfg, rank, world);
  if (rc) return rc;
  EP_ARG(nccl_uid != nullptr || !(cfg->transports & DYMOE_EP_NCCL),
         "nccl_uid: required when cfg.transports includes DYMOE_EP_NCCL");
  dymoe_ep* ep = new (std::nothrow) dymoe_ep();
  if (!ep) return fail(DYMOE_ERR_INVALID, "out of host memory");
  ep->rank = rank;
  ep->P = world;
  ep->M = cfg->M;
  ep->k = cfg->k_route;
  ep->Hd = cfg->hidden;
  ep->F = cfg->ffn;
  ep->max_T = cfg->max_tokens;
  ep->cap = cfg->max_tokens * cfg->k_route * world;
  ep->transports = cfg->transports;
  ep->first = ep_first_of_owner(rank, cfg->M, world);
  ep->last = ep_first_of_owner(rank + 1, cfg->M, world);
  auto bail = [&](int code) {
    destroy(ep);
    return code;
  };
  // every kernel loaded before any peer can spin in a barrier (include/dymoe.h dymoe_preload)
  rc = dymoe_preload();
  if (rc) return bail(rc);
  ep->win_bytes = ep_win_layout(world, cfg->M, cfg->hidden, ep->cap).total;
  cudaError_t e = cudaMalloc(&ep->win, ep->win_bytes);
  if (e == cudaSuccess) e = cudaMemset(ep->win, 0, ep->win_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&ep->peers_dev, sizeof(char*) * world);
  if (e == cudaSuccess) e = cudaMalloc(&ep->self_dev, sizeof(char*));
  if (e == cudaSuccess) e = cudaMemcpy(ep->self_dev, &ep->win, sizeof(char*), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&ep->ident, sizeof(int32_t) * ep->cap);
  if (e == cudaSuccess) {
    k_iota<<<256, 256>>>(ep->ident, ep->cap);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMallocHost(&ep->host_cnt, sizeof(int32_t) * world * cfg->M);
  if (e == cudaSuccess) e = cudaMallocHost(&ep->host_roff, sizeof(int32_t) * (cfg->M + 1));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(DYMOE_ERR_CUDA, "dymoe_ep_create: %s", cudaGetErrorString(e)));
  if (world == 1) {   // a single rank is its own only peer
    void* b = ep->win;
    rc = do_connect(ep, &b);
    if (rc) return bail(rc);
  }
  if (nccl_uid != nullptr) {
    const NcclApi& N = nccl();
    if (!N.ok) return bail(fail(DYMOE_ERR_NCCL, "%s", N.why));
    ncclUniqueId id;
    memcpy(&id, nccl_uid, sizeof(id));
    ncclResult_t r = N.CommInitRank(&ep->comm, world, id, rank);
    if (r != ncclSuccess) {
      ep->comm = nullptr;
      return bail(fail(DYMOE_ERR_NCCL, "ncclCommInitRank: %s", N.GetErrorString(r)));
    }
    if ((cfg->transports & DYMOE_EP_PEER) && world > 1) {
      // windows over the communicator: all-gather the IPC handles, open the peers'
      cudaIpcMemHandle_t mine;
      e = cudaIpcGetMemHandle(&mine, ep->win);
      if (e != cudaSuccess) return bail(fail(DYMOE_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e)));
      char* dev = nullptr;
      e = cudaMalloc(&dev, (size_t)(world + 1) * sizeof(mine));
      if (e == cudaSuccess) e = cudaMemcpy(dev, &mine, sizeof(mine), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        cudaFree(dev);
        return bail(fail(DYMOE_ERR_CUDA, "dymoe_ep_create: %s", cudaGetErrorString(e)));
      }
      r = N.AllGather(dev, dev + sizeof(mine), sizeof(mine), ncclUint8, ep->comm, nullptr);
      std::vector<cudaIpcMemHandle_t> all(world);
      if (r == ncclSuccess) e = cudaMemcpy(all.data(), dev + sizeof(mine), sizeof(mine) * world, cudaMemcpyDeviceToHost);
      cudaFree(dev);
      if (r != ncclSuccess) return bail(fail(DYMOE_ERR_NCCL, "ncclAllGather(ipc handles): %s", N.GetErrorString(r)));
      if (e != cudaSuccess) return bail(fail(DYMOE_ERR_CUDA, "dymoe_ep_create: %s", cudaGetErrorString(e)));
      std::vector<void*> bases(world);
      for (int p = 0; p < world; ++p) {
        if (p == rank) {
          bases[p] = ep->win;
          continue;
        }
        e = cudaIpcOpenMemHandle(&bases[p], all[p], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return bail(fail(DYMOE_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", p, cudaGetErrorString(e)));
        ep->opened.push_back(bases[p]);
      }
      rc = do_connect(ep, bases.data());
      if (rc) return bail(rc);
    }
  }
  *out = ep;
  clear_error();
  return DYMOE_OK;
}

int dymoe_ep_window_base(const dymoe_ep* ep, void** base, void* ipc_handle) {
  EP_ARG(ep != nullptr, "ep: must not be NULL");
  EP_ARG(base != nullptr, "base: must not be NULL");
  *base = ep->win;
  if (ipc_handle != nullptr) {
    cudaIpcMemHandle_t h;
    EP_CUDA(cudaIpcGetMemHandle(&h, ep->win), "dymoe_ep_window_base");
    memcpy(ipc_handle, &h, sizeof(h));
  }
  clear_error();
  return DYMOE_OK;
}

int dymoe_ep_connect(dymoe_ep* ep, void* const* peer_bases) {
  EP_ARG(ep != nullptr, "ep: must not be NULL");
  EP_ARG(peer_bases != nullptr, "peer_bases: must not be NULL");
  const int rc = do_connect(ep, peer_bases);
  if (rc) return rc;
  clear_error();
  return DYMOE_OK;
}

size_t dymoe_ep_workspace_size(const dymoe_ep* ep, int T, int T_peer_max, int placement) {
  if (ep == nullptr || T < 0) return 0;
  return ep_ws(ep, T, T_peer_max, placement).total;
}

int dymoe_ep_workspace_views(const dymoe_ep* ep, int T, int T_peer_max, int placement,
                             void* ws, dymoe_ws_views* v) {
  EP_ARG(ep != nullptr, "ep: must not be NULL");
  EP_ARG(ws != nullptr, "workspace: must not be NULL");
  EP_ARG(v != nullptr, "views: must not be NULL");
  const EpWs W = ep_ws(ep, T, T_peer_max, placement);
  memset(v, 0, sizeof(*v));
  v->topk_idx = at<int32_t>(ws, W.topk_idx);
  v->topk_w = at<float>(ws, W.topk_w);
  v->probs = at<float>(ws, W.probs);
  v->importance = at<float>(ws, W.imp);
  v->heavy = at<int32_t>(ws, W.heavy);
  v->bits = at<uint8_t>(ws, W.bits);
  v->active = at<uint8_t>(ws, W.active);
  v->expert_off = at<int32_t>(ws, W.off);
  v->perm_token = at<int32_t>(ws, W.perm_token);
  v->perm_slot = at<int32_t>(ws, W.perm_slot);
  v->inv_row = at<int32_t>(ws, W.inv_row);
  v->status = at<uint32_t>(ws, W.status);
  v->score_scratch = at<void>(ws, W.score_scratch);
  clear_error();
  return DYMOE_OK;
}

int dymoe_moe_forward_ep(dymoe_ep* ep, const dymoe_layer* local, int transport, int placement,
                         const uint16_t* x, const float* logits, int T, int T_peer_max,
                         const dymoe_fwd_opts* o, void* y, void* ws, size_t ws_bytes,
                         dymoe_stream_t stream) {
  EP_ARG(ep != nullptr, "ep: must not be NULL");
  EP_ARG(o != nullptr, "opts: must not be NULL");
  EP_ARG(transport == DYMOE_EP_NCCL || transport == DYMOE_EP_PEER,
         "transport: must be DYMOE_EP_NCCL or DYMOE_EP_PEER");
  EP_ARG(ep->transports & transport, "transport: not enabled in cfg.transports at dymoe_ep_create");
  EP_ARG(transport != DYMOE_EP_NCCL || ep->comm != nullptr, "transport: the handle has no communicator");
  EP_ARG(transport != DYMOE_EP_PEER || ep->connected, "transport: windows not connected (dymoe_ep_connect)");
  EP_ARG(placement == DYMOE_EP_ALL_TO_ALL || placement == DYMOE_EP_REPLICATED,
         "placement: must be DYMOE_EP_ALL_TO_ALL or DYMOE_EP_REPLICATED");
  EP_ARG(T >= 0 && T <= ep->max_T, "T: must satisfy 0 <= T <= cfg.max_tokens (%d)", ep->max_T);
  EP_ARG(T_peer_max == 0 || (T_peer_max >= T && T_peer_max <= ep->max_T),
         "T_peer_max: must be 0 or in [T, cfg.max_tokens]");
  const int M_loc = ep->last - ep->first;
  if (M_loc > 0) {
    EP_ARG(local != nullptr, "local: must not be NULL on a rank that owns experts");
    EP_ARG(local->M == M_loc, "local.M: %d, but this rank owns %d experts", local->M, M_loc);
    EP_ARG(local->k == 1, "local.k_route: must be 1 (a table of owned experts)");
    EP_ARG(local->Hd == ep->Hd && local->F == ep->F, "local: hidden / ffn differ from cfg");
  }
  EP_ARG(o->phase == DYMOE_PREFILL || o->phase == DYMOE_DECODE, "opts.phase: must be DYMOE_PREFILL or DYMOE_DECODE");
  EP_ARG(o->out_dtype == DYMOE_OUT_F32 || o->out_dtype == DYMOE_OUT_BF16,
         "opts.out_dtype: must be DYMOE_OUT_F32 or DYMOE_OUT_BF16");
  EP_ARG(o->ffn_mode == -1 || o->ffn_mode == DYMOE_PREFILL || o->ffn_mode == DYMOE_DECODE,
         "opts.ffn_mode: must be -1, DYMOE_PREFILL or DYMOE_DECODE");
  AssignParams ap{};
  int rc = assign_params(&o->ladder, ep->M, ep->k, o->layer, o->num_layers, ap);
  if (rc) return rc;
  int k_tokens = o->k_tokens;
  if (placement == DYMOE_EP_REPLICATED) {
    EP_ARG(o->phase == DYMOE_DECODE, "opts.phase: DYMOE_EP_REPLICATED is a decode placement");
    EP_ARG(T <= kEpRedRows, "T: DYMOE_EP_REPLICATED takes at most %d tokens", kEpRedRows);
  } else if (o->phase == DYMOE_PREFILL && T > 0) {
    EP_ARG(o->attn_mass != nullptr, "opts.attn_mass: must not be NULL in PREFILL");
    EP_ARG(o->heads >= 1, "opts.heads: must be >= 1");
    if (k_tokens == 0) k_tokens = (T + 4) / 5;
    EP_ARG(k_tokens >= 0 && k_tokens <= T, "opts.k_tokens: must satisfy 0 <= k_tokens <= T");
  }
  EP_ARG(ws != nullptr, "workspace: must not be NULL");
  EP_ARG(((uintptr_t)ws % 256) == 0, "workspace: must be 256-byte aligned");
  EP_ARG(T == 0 || (x != nullptr && logits != nullptr && y != nullptr), "x/logits/y: must not be NULL");
  EP_ARG(((uintptr_t)x % 16) == 0, "x: must be 16-byte aligned");
  const EpWs W = ep_ws(ep, T, T_peer_max, placement);
  if (ws_bytes < W.total)
    return fail(DYMOE_ERR_WORKSPACE, "ws_bytes: %zu < dymoe_ep_workspace_size() = %zu", ws_bytes, W.total);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (T > 0)
    EP_CUDA(launch_route(logits, T, ep->M, ep->k, at<int32_t>(ws, W.topk_idx), at<float>(ws, W.topk_w),
                         at<float>(ws, W.probs), s),
            "route");
  if (placement == DYMOE_EP_REPLICATED) {
    if (T == 0) return DYMOE_OK;   // every rank has the same batch: nothing to exchange
    rc = replicated(ep, local, transport, o, ap, x, logits, T, y, ws, W, s);
  } else if (transport == DYMOE_EP_PEER) {
    rc = a2a_peer(ep, local, o, ap, x, logits, T, y, ws, W, k_tokens, s);
  } else {
    rc = a2a_nccl(ep, local, o, ap, x, logits, T, y, ws, W, k_tokens, s);
  }
  if (rc) return rc;
  clear_error();
  return DYMOE_OK;
}

int dymoe_ep_check_status(const dymoe_ep* ep, int T, int T_peer_max, int placement, void* ws,
                          uint32_t* bits_out, dymoe_stream_t stream) {
  EP_ARG(ep != nullptr, "ep: must not be NULL");
  EP_ARG(ws != nullptr, "workspace: must not be NULL");
  const EpWs W = ep_ws(ep, T, T_peer_max, placement);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint32_t word = 0;
  EP_CUDA(cudaMemcpyAsync(&word, at<uint32_t>(ws, W.status), 4, cudaMemcpyDeviceToHost, s), "status");
  EP_CUDA(cudaStreamSynchronize(s), "status");
  EP_CUDA(cudaMemsetAsync(at<uint32_t>(ws, W.status), 0, 4, s), "status");
  if (bits_out) *bits_out = word;
  if (word)
    return fail(DYMOE_ERR_DEVICE, "device status word 0x%x (1: width not resident, 2: barrier timeout, 4: window overflow)", word);
  clear_error();
  return DYMOE_OK;
}

int dymoe_ep_destroy(dymoe_ep* ep) {
  destroy(ep);
  clear_error();
  return DYMOE_OK;
}

}  // extern "C"

cudaError_t dymoe::preload_ep_layer() {
  return preload_kernels(k_counts_from_off, k_route_hist, k_active_from_counts, k_local_view, k_iota);
}
