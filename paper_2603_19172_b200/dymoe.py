"""Thin ctypes binding over libdymoe.so (include/dymoe.h).

Argument marshalling only: every step of the path runs in the library's CUDA kernels.  torch
is used for device memory (output allocation) and streams.  There is no CPU fallback: if the
library is missing or the tensors are not on a CUDA device the calls raise.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdymoe.so")

DYMOE_OK = 0
DYMOE_PREFILL, DYMOE_DECODE = 0, 1
DYMOE_M_TOTAL, DYMOE_M_ACTIVE = 0, 1
DYMOE_OUT_F32, DYMOE_OUT_BF16 = 0, 1
MAX_TIERS = 5
GROUP = 128
WIDTH_INDEX = {8: 0, 4: 1, 2: 2}

EXPORTED = [
    "dymoe_route", "dymoe_score", "dymoe_score_scratch_bytes", "dymoe_assign_bits",
    "dymoe_retention_ratio", "dymoe_tier_counts", "dymoe_quantize", "dymoe_quantize_batched",
    "dymoe_layer_create", "dymoe_layer_refresh", "dymoe_layer_destroy", "dymoe_permute", "dymoe_expert_ffn",
    "dymoe_combine", "dymoe_workspace_size", "dymoe_workspace_views", "dymoe_moe_forward",
    "dymoe_check_status", "dymoe_last_error", "dymoe_version", "dymoe_ep_plan",
    "dymoe_gather_rows", "dymoe_renorm_weights", "dymoe_predict_ws_bytes", "dymoe_predict_next",
    "dymoe_pool_create", "dymoe_pool_destroy", "dymoe_pool_lookup", "dymoe_pool_insert",
    "dymoe_pool_pin", "dymoe_pool_unpin", "dymoe_pool_snapshot", "dymoe_pool_used",
    "dymoe_layer_set_expert", "dymoe_attention_mass", "dymoe_gate_logits",
    "dymoe_rmsnorm", "dymoe_ep_window_bytes", "dymoe_ep_window_alloc", "dymoe_ep_window_open",
    "dymoe_ep_window_close", "dymoe_ep_window_free", "dymoe_ep_publish_counts", "dymoe_ep_barrier",
    "dymoe_ep_dispatch", "dymoe_ep_combine", "dymoe_preload", "dymoe_permute_scratch_bytes",
    "dymoe_expert_ffn_ws_bytes", "dymoe_ep_unique_id", "dymoe_ep_create", "dymoe_ep_window_base",
    "dymoe_ep_connect", "dymoe_ep_workspace_size", "dymoe_ep_workspace_views",
    "dymoe_moe_forward_ep", "dymoe_ep_check_status", "dymoe_ep_destroy", "dymoe_ep_plan_host",
]
DYMOE_EP_NCCL, DYMOE_EP_PEER = 1, 2
DYMOE_EP_ALL_TO_ALL, DYMOE_EP_REPLICATED = 0, 1
EP_UID_BYTES, EP_IPC_BYTES = 128, 64
DYMOE_STATUS_EP_TIMEOUT, DYMOE_STATUS_EP_OVERFLOW = 2, 4


class DymoeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("dymoe error %d: %s" % (code, msg))
        self.code = code
        self.msg = msg


class Ladder(ctypes.Structure):
    _fields_ = [("n_tiers", ctypes.c_int), ("bits", ctypes.c_int * MAX_TIERS),
                ("lambdas", ctypes.c_double * (MAX_TIERS - 1)), ("clamp_to_k", ctypes.c_int),
                ("m_mode", ctypes.c_int), ("renorm_on_skip", ctypes.c_int)]


class QuantJob(ctypes.Structure):
    _fields_ = [("W", ctypes.c_void_p), ("N", ctypes.c_int), ("K", ctypes.c_int),
                ("bits", ctypes.c_int), ("codes", ctypes.c_void_p), ("scales", ctypes.c_void_p),
                ("zeros", ctypes.c_void_p)]


class QMat(ctypes.Structure):
    _fields_ = [("codes", ctypes.c_void_p), ("scales", ctypes.c_void_p), ("zeros", ctypes.c_void_p)]


class ExpertDesc(ctypes.Structure):
    _fields_ = [("w1", ctypes.c_void_p), ("w3", ctypes.c_void_p), ("w2", ctypes.c_void_p),
                ("q", (QMat * 3) * 3)]


class LayerDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int), ("k_route", ctypes.c_int), ("hidden", ctypes.c_int),
                ("ffn", ctypes.c_int), ("experts", ctypes.POINTER(ExpertDesc))]


class FwdOpts(ctypes.Structure):
    _fields_ = [("phase", ctypes.c_int), ("layer", ctypes.c_int), ("num_layers", ctypes.c_int),
                ("ladder", Ladder), ("attn_mass", ctypes.c_void_p), ("heads", ctypes.c_int),
                ("k_tokens", ctypes.c_int), ("ffn_mode", ctypes.c_int), ("out_dtype", ctypes.c_int),
                ("forced_bits", ctypes.c_void_p), ("prof_events", ctypes.c_void_p * 3),
                ("residual", ctypes.c_void_p)]


class WsViews(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "topk_idx", "topk_w", "probs", "importance", "heavy", "bits", "active", "expert_off",
        "perm_token", "perm_slot", "inv_row", "h", "y_perm", "status", "score_scratch")]


_lib = None


class EpConfig(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int), ("k_route", ctypes.c_int), ("hidden", ctypes.c_int),
                ("ffn", ctypes.c_int), ("max_tokens", ctypes.c_int), ("transports", ctypes.c_int)]


class EpWindow(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int), ("rank", ctypes.c_int), ("M", ctypes.c_int), ("Hd", ctypes.c_int),
                ("cap_rows", ctypes.c_int), ("parity", ctypes.c_int), ("peers", ctypes.c_void_p)]


def lib():
    """Load libdymoe.so once; raise loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libdymoe.so not built at %s (run paper_2603_19172_b200.build)" % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        vp, ci, cz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        sig = {
            "dymoe_route": [vp, ci, ci, ci, vp, vp, vp, vp],
            "dymoe_score": [ci, vp, ci, vp, vp, ci, ci, ci, ci, vp, vp, vp, vp],
            "dymoe_score_scratch_bytes": [ci],
            "dymoe_assign_bits": [vp, ci, ci, ci, ctypes.POINTER(Ladder), ci, vp, vp, vp, vp],
            "dymoe_retention_ratio": [ci, ci, ctypes.c_double],
            "dymoe_tier_counts": [ci, ci, ctypes.POINTER(Ladder), ci, ci, vp],
            "dymoe_quantize": [vp, ci, ci, ci, ci, vp, vp, vp, vp],
            "dymoe_quantize_batched": [ctypes.POINTER(QuantJob), ci, ci, vp],
            "dymoe_layer_create": [ctypes.POINTER(LayerDesc), ctypes.POINTER(vp)],
            "dymoe_layer_destroy": [vp],
            "dymoe_layer_refresh": [vp, vp],
            "dymoe_permute": [vp, ci, ci, ci, vp, vp, vp, vp, vp, vp, cz, vp],
            "dymoe_permute_scratch_bytes": [ci, ci, ci],
            "dymoe_expert_ffn": [vp, ci, vp, ci, vp, vp, vp, vp, vp, vp, vp, cz, vp],
            "dymoe_expert_ffn_ws_bytes": [vp, ci],
            "dymoe_combine": [vp, vp, vp, ci, ci, ci, ci, ci, vp, vp],
            "dymoe_workspace_size": [vp, ci],
            "dymoe_workspace_views": [vp, ci, vp, ctypes.POINTER(WsViews)],
            "dymoe_moe_forward": [vp, vp, vp, ci, ctypes.POINTER(FwdOpts), vp, vp, cz, vp],
            "dymoe_check_status": [vp, ci, vp, vp, vp],
            "dymoe_last_error": [],
            "dymoe_version": [],
            "dymoe_ep_plan": [vp, ci, ci, vp, vp, vp],
            "dymoe_gather_rows": [vp, ci, vp, ci, vp, vp],
            "dymoe_renorm_weights": [vp, vp, vp, ci, ci, ci, ci, vp, vp],
            "dymoe_predict_ws_bytes": [ci, ci, ci],
            "dymoe_predict_next": [ci, vp, vp, ci, ci, ci, ci, ci, vp, cz, vp, vp, vp, vp, vp],
            "dymoe_pool_create": [cz, ctypes.POINTER(vp)],
            "dymoe_pool_destroy": [vp],
            "dymoe_pool_lookup": [vp, ci, ci, ci, ctypes.POINTER(ci), ctypes.POINTER(ci),
                                  ctypes.POINTER(cz)],
            "dymoe_pool_insert": [vp, ci, ci, ci, cz, ctypes.POINTER(cz), vp, ci, ctypes.POINTER(ci)],
            "dymoe_pool_pin": [vp, ci, ci],
            "dymoe_pool_unpin": [vp, ci, ci],
            "dymoe_pool_snapshot": [vp, vp, ci, ctypes.POINTER(ci)],
            "dymoe_pool_used": [vp],
            "dymoe_layer_set_expert": [vp, ci, ctypes.POINTER(ExpertDesc), vp],
            "dymoe_attention_mass": [vp, vp, ci, ci, ci, ctypes.c_float, vp, vp, vp],
            "dymoe_gate_logits": [vp, vp, vp, ci, ci, ci, vp, vp],
            "dymoe_rmsnorm": [vp, ci, ci, ctypes.c_float, vp, vp],
            "dymoe_ep_window_bytes": [ci, ci, ci, ci],
            "dymoe_preload": [],
            "dymoe_ep_window_alloc": [cz, ctypes.POINTER(vp), vp],
            "dymoe_ep_window_open": [vp, ctypes.POINTER(vp)],
            "dymoe_ep_window_close": [vp],
            "dymoe_ep_window_free": [vp],
            "dymoe_ep_publish_counts": [ctypes.POINTER(EpWindow), vp, vp],
            "dymoe_ep_barrier": [ctypes.POINTER(EpWindow), ctypes.c_uint32, vp, vp],
            "dymoe_ep_dispatch": [ctypes.POINTER(EpWindow), vp, ci, vp, vp, vp, vp, vp],
            "dymoe_ep_combine": [ctypes.POINTER(EpWindow), vp, vp, ci, ci, vp, ci, ci, vp, vp, vp],
            "dymoe_ep_unique_id": [vp],
            "dymoe_ep_create": [ci, ci, vp, ctypes.POINTER(EpConfig), ctypes.POINTER(vp)],
            "dymoe_ep_window_base": [vp, ctypes.POINTER(vp), vp],
            "dymoe_ep_connect": [vp, vp],
            "dymoe_ep_workspace_size": [vp, ci, ci, ci],
            "dymoe_ep_workspace_views": [vp, ci, ci, ci, vp, ctypes.POINTER(WsViews)],
            "dymoe_moe_forward_ep": [vp, vp, ci, ci, vp, vp, ci, ci, ctypes.POINTER(FwdOpts), vp, vp,
                                     cz, vp],
            "dymoe_ep_check_status": [vp, ci, ci, ci, vp, vp, vp],
            "dymoe_ep_destroy": [vp],
            "dymoe_ep_plan_host": [ci, ci, ci, vp, vp, vp, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ci
        L.dymoe_retention_ratio.restype = ctypes.c_double
        L.dymoe_score_scratch_bytes.restype = cz
        L.dymoe_workspace_size.restype = cz
        L.dymoe_predict_ws_bytes.restype = cz
        L.dymoe_pool_used.restype = cz
        L.dymoe_ep_window_bytes.restype = cz
        L.dymoe_permute_scratch_bytes.restype = cz
        L.dymoe_expert_ffn_ws_bytes.restype = cz
        L.dymoe_ep_workspace_size.restype = cz
        L.dymoe_last_error.restype = ctypes.c_char_p
        L.dymoe_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc):
    if rc != DYMOE_OK:
        raise DymoeError(rc, lib().dymoe_last_error().decode())


def _p(t):
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("dymoe: tensors must live on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("dymoe: tensors must be contiguous")
    return t.data_ptr()


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _u16(t):
    """bf16 tensor viewed as its bit patterns (no copy)."""
    return t.view(torch.int16) if t.dtype == torch.bfloat16 else t


def make_ladder(bits, lambdas, clamp_to_k=True, m_active=False, renorm_on_skip=True):
    L = Ladder()
    L.n_tiers = len(bits)
    for i, b in enumerate(bits):
        L.bits[i] = int(b)
    for i, lam in enumerate(lambdas):
        L.lambdas[i] = float(lam)
    L.clamp_to_k = int(bool(clamp_to_k))
    L.m_mode = DYMOE_M_ACTIVE if m_active else DYMOE_M_TOTAL
    L.renorm_on_skip = int(bool(renorm_on_skip))
    return L


# ---------------------------------------------------------------------------------------------
def dymoe_route(logits, k, with_probs=True, stream=None):
    T, M = logits.shape
    dev = logits.device
    idx = torch.empty(T, k, dtype=torch.int32, device=dev)
    w = torch.empty(T, k, dtype=torch.float32, device=dev)
    p = torch.empty(T, M, dtype=torch.float32, device=dev) if with_probs else None
    _check(lib().dymoe_route(_p(logits), T, M, k, _p(idx), _p(w), _p(p), _stream(stream)))
    return idx, w, p


def dymoe_score(phase, M, k=0, topk_idx=None, attn_mass=None, logits=None, k_tokens=0,
                stream=None):
    if phase == DYMOE_PREFILL:
        H, T = attn_mass.shape
        dev = attn_mass.device
    else:
        T = logits.shape[0]
        H = 0
        dev = logits.device
    imp = torch.empty(M, dtype=torch.float32, device=dev)
    kt = k_tokens if k_tokens else (T + 4) // 5
    heavy = torch.full((max(kt, 1),), -1, dtype=torch.int32, device=dev) if phase == DYMOE_PREFILL else None
    scratch = torch.empty(lib().dymoe_score_scratch_bytes(T), dtype=torch.uint8, device=dev) \
        if phase == DYMOE_PREFILL else None
    _check(lib().dymoe_score(phase, _p(attn_mass), H, _p(topk_idx), _p(logits), T, M, k, k_tokens,
                             _p(imp), _p(heavy), _p(scratch), _stream(stream)))
    return imp, (heavy[:kt] if heavy is not None else None)


def dymoe_assign_bits(importance, layer, num_layers, ladder, k_route, active_mask=None,
                      stream=None):
    M = importance.shape[0]
    bits = torch.empty(M, dtype=torch.uint8, device=importance.device)
    counts = (ctypes.c_int32 * MAX_TIERS)()
    _check(lib().dymoe_assign_bits(_p(importance), M, layer, num_layers, ctypes.byref(ladder),
                                   k_route, _p(active_mask), _p(bits), ctypes.cast(counts, ctypes.c_void_p),
                                   _stream(stream)))
    return bits, [counts[i] for i in range(ladder.n_tiers - 1)]


def dymoe_retention_ratio(layer, num_layers, lam):
    return lib().dymoe_retention_ratio(layer, num_layers, lam)


def dymoe_tier_counts(layer, num_layers, ladder, M_eff, k_route):
    counts = (ctypes.c_int32 * MAX_TIERS)()
    _check(lib().dymoe_tier_counts(layer, num_layers, ctypes.byref(ladder), M_eff, k_route,
                                   ctypes.cast(counts, ctypes.c_void_p)))
    return [counts[i] for i in range(ladder.n_tiers - 1)]


def alloc_qmat(N, K, bits, device):
    codes = torch.empty(N, K * bits // 32, dtype=torch.int32, device=device)
    scales = torch.empty(N, K // GROUP, dtype=torch.float32, device=device)
    zeros = torch.empty(N, K // GROUP, dtype=torch.uint8, device=device)
    return codes, scales, zeros


def dymoe_quantize(W, bits, out=None, stream=None):
    N, K = W.shape
    codes, scales, zeros = out if out is not None else alloc_qmat(N, K, bits, W.device)
    _check(lib().dymoe_quantize(_p(_u16(W)), N, K, bits, GROUP, _p(codes), _p(scales), _p(zeros),
                                _stream(stream)))
    return codes, scales, zeros


def dymoe_quantize_batched(jobs, stream=None):
    """jobs: list of (W bf16 [N,K], bits, (codes, scales, zeros))."""
    arr = (QuantJob * max(len(jobs), 1))()
    for i, (W, bits, (c, s, z)) in enumerate(jobs):
        arr[i] = QuantJob(_p(_u16(W)), W.shape[0], W.shape[1], bits, _p(c), _p(s), _p(z))
    _check(lib().dymoe_quantize_batched(arr, len(jobs), GROUP, _stream(stream)))


def dymoe_permute(topk_idx, M, bits, stream=None):
    T, k = topk_idx.shape
    dev = topk_idx.device
    off = torch.empty(M + 1, dtype=torch.int32, device=dev)
    pt = torch.empty(max(T * k, 1), dtype=torch.int32, device=dev)
    ps = torch.empty(max(T * k, 1), dtype=torch.int32, device=dev)
    inv = torch.empty(T, k, dtype=torch.int32, device=dev)
    nb = lib().dymoe_permute_scratch_bytes(T, k, M)
    scratch = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
    _check(lib().dymoe_permute(_p(topk_idx), T, k, M, _p(bits), _p(off), _p(pt), _p(ps), _p(inv),
                               _p(scratch), scratch.numel(), _stream(stream)))
    return off, pt, ps, inv


def dymoe_ep_plan(expert_off, P, stream=None):
    """(send_counts int32 [P], row_expert int32 [rows]) for expert-parallel dispatch."""
    M = expert_off.shape[0] - 1
    dev = expert_off.device
    sc = torch.empty(P, dtype=torch.int32, device=dev)
    R = int(expert_off[-1].item()) if expert_off.is_cuda else int(expert_off[-1])
    re = torch.empty(max(R, 1), dtype=torch.int32, device=dev)
    _check(lib().dymoe_ep_plan(_p(expert_off), M, P, _p(sc), _p(re), _stream(stream)))
    return sc, re[:R]


def dymoe_gather_rows(x, rows, stream=None):
    n = rows.shape[0]
    out = torch.empty(n, x.shape[1], dtype=x.dtype, device=x.device)
    _check(lib().dymoe_gather_rows(_p(_u16(x)), x.shape[1], _p(rows), n, _p(_u16(out)) if n else None,
                                   _stream(stream)))
    return out


def dymoe_ep_window_bytes(P, M, Hd, cap_rows):
    return lib().dymoe_ep_window_bytes(P, M, Hd, cap_rows)


def dymoe_ep_window_alloc(nbytes):
    """(base pointer int, 64-byte CUDA IPC handle) of a zeroed device window (caller frees)."""
    base = ctypes.c_void_p()
    h = ctypes.create_string_buffer(64)
    _check(lib().dymoe_ep_window_alloc(nbytes, ctypes.byref(base), h))
    return base.value, bytes(h.raw)


def dymoe_ep_window_open(handle):
    base = ctypes.c_void_p()
    _check(lib().dymoe_ep_window_open(ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(base)))
    return base.value


def dymoe_ep_window_close(base):
    _check(lib().dymoe_ep_window_close(ctypes.c_void_p(base)))


def dymoe_ep_window_free(base):
    _check(lib().dymoe_ep_window_free(ctypes.c_void_p(base)))


def dymoe_ep_publish_counts(win, expert_off, stream=None):
    _check(lib().dymoe_ep_publish_counts(ctypes.byref(win), _p(expert_off), _stream(stream)))


def dymoe_ep_barrier(win, epoch, status=None, stream=None):
    _check(lib().dymoe_ep_barrier(ctypes.byref(win), epoch & 0xffffffff, _p(status), _stream(stream)))


def dymoe_ep_dispatch(win, x, expert_off, perm_token, recv_off, status=None, stream=None):
    _check(lib().dymoe_ep_dispatch(ctypes.byref(win), _p(_u16(x)), x.shape[0], _p(expert_off),
                                   _p(perm_token), _p(recv_off), _p(status), _stream(stream)))


def dymoe_ep_combine(win, inv_row, topk_w, expert_off, renorm=True, out_dtype=DYMOE_OUT_F32,
                     status=None, stream=None):
    T, k = inv_row.shape
    y = torch.empty(T, win.Hd, dtype=torch.float32 if out_dtype == DYMOE_OUT_F32 else torch.bfloat16,
                    device=inv_row.device)
    _check(lib().dymoe_ep_combine(ctypes.byref(win), _p(inv_row), _p(topk_w), T, k, _p(expert_off),
                                  int(renorm), out_dtype, _p(y) if T else None, _p(status),
                                  _stream(stream)))
    return y


def dymoe_ep_plan_host(P, M, rank, counts):
    """Host-side all-to-all plan (include/dymoe.h): counts int32 [P][M] (CPU) ->
    (send_off int64 [M+1], recv_base int64 [M_loc][P], recv_off int32 [M_loc+1]).  No GPU."""
    counts = torch.as_tensor(counts, dtype=torch.int32).contiguous()
    first = -(-rank * M // P)
    last = -(-(rank + 1) * M // P)
    m_loc = last - first
    so = torch.empty(M + 1, dtype=torch.int64)
    rb = torch.empty(max(m_loc * P, 1), dtype=torch.int64)
    ro = torch.empty(m_loc + 1, dtype=torch.int32)
    _check(lib().dymoe_ep_plan_host(P, M, rank, counts.data_ptr(), so.data_ptr(), rb.data_ptr(),
                                    ro.data_ptr()))
    return so, rb[:m_loc * P].view(m_loc, P), ro


def dymoe_combine(y_perm, inv_row, topk_w, renorm=True, out_dtype=DYMOE_OUT_F32, stream=None):
    T, k = inv_row.shape
    Hd = y_perm.shape[1]
    y = torch.empty(T, Hd, dtype=torch.float32 if out_dtype == DYMOE_OUT_F32 else torch.bfloat16,
                    device=y_perm.device)
    _check(lib().dymoe_combine(_p(y_perm), _p(inv_row), _p(topk_w), T, k, Hd, int(renorm),
                               out_dtype, _p(y), _stream(stream)))
    return y


def dymoe_attention_mass(q, k, scale=None, stream=None):
    """Causal attention mass a [H][T] f32 from q, k [H][T][d] bf16 (include/dymoe.h)."""
    H, T, dd = q.shape
    scale = dd ** -0.5 if scale is None else scale
    scratch = torch.empty(2 * H * T, dtype=torch.float32, device=q.device)
    a = torch.empty(H, T, dtype=torch.float32, device=q.device)
    _check(lib().dymoe_attention_mass(_p(_u16(q)), _p(_u16(k)), H, T, dd, float(scale), _p(scratch),
                                      _p(a), _stream(stream)))
    return a


def dymoe_renorm_weights(topk_idx, topk_w, bits, renorm=True, stream=None):
    """Combine weights against the global live set (D12; include/dymoe.h)."""
    T, k = topk_idx.shape
    out = torch.empty_like(topk_w)
    _check(lib().dymoe_renorm_weights(_p(topk_idx), _p(topk_w), _p(bits), T, k, bits.shape[0],
                                      int(renorm), _p(out), _stream(stream)))
    return out


def dymoe_rmsnorm(x, eps=1e-5, out=None, stream=None):
    """u [T][Hd] bf16 = bf16(x / sqrt(mean(x^2) + eps)), x bf16 [T][Hd]."""
    T, Hd = x.shape
    u = out if out is not None else torch.empty_like(x)
    _check(lib().dymoe_rmsnorm(_p(_u16(x)), T, Hd, eps, _p(_u16(u)), _stream(stream)))
    return u


def dymoe_gate_logits(h, w_gate, bias=None, out=None, stream=None):
    """logits [T][M] f32 = h [T][Hd] bf16 . w_gate [M][Hd] bf16 (fp32, error bound of reading P1) + bias [M]."""
    T, Hd = h.shape
    M = w_gate.shape[0]
    lg = out if out is not None else torch.empty(T, M, dtype=torch.float32, device=h.device)
    _check(lib().dymoe_gate_logits(_p(_u16(h)), _p(_u16(w_gate)), _p(bias), T, Hd, M, _p(lg),
                                   _stream(stream)))
    return lg


def dymoe_predict_next(phase, h, w_gate_next, k_route, t, stream=None):
    """Eqs. 6-8 look-ahead (include/dymoe.h).  Returns (experts [n] i32, priority [n] f32,
    logits [T][M] f32) on the device; n = number of valid requests (one host read)."""
    T, Hd = h.shape
    M = w_gate_next.shape[0]
    nbytes = lib().dymoe_predict_ws_bytes(T, M, k_route)
    ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=h.device)
    ex = torch.empty(t, dtype=torch.int32, device=h.device)
    pr = torch.empty(t, dtype=torch.float32, device=h.device)
    n = torch.empty(1, dtype=torch.int32, device=h.device)
    lg = torch.empty(T, M, dtype=torch.float32, device=h.device)
    _check(lib().dymoe_predict_next(phase, _p(_u16(h)), _p(_u16(w_gate_next)), T, Hd, M, k_route, t,
                                    _p(ws), ws.numel(), _p(ex), _p(pr), _p(n), _p(lg), _stream(stream)))
    k = int(n.item())
    return ex[:k], pr[:k], lg


def _fill_desc(d, ex):
    for n in ("w1", "w3", "w2"):
        t = ex.get(n)
        setattr(d, n, _p(_u16(t)) if t is not None else None)
    for b, wi in WIDTH_INDEX.items():
        q = ex.get("q%d" % b)
        if q is None:
            continue
        for mi, n in enumerate(("w1", "w3", "w2")):
            c, s_, z = q[n]
            d.q[wi][mi] = QMat(_p(c), _p(s_), _p(z))


# ---------------------------------------------------------------------------------------------
class PoolEntry(ctypes.Structure):
    _fields_ = [("layer", ctypes.c_int), ("expert", ctypes.c_int), ("bits", ctypes.c_int),
                ("pins", ctypes.c_int), ("bytes", ctypes.c_size_t), ("offset", ctypes.c_size_t),
                ("last_use", ctypes.c_ulonglong)]


POOL_HIT, POOL_MISS, POOL_PROMOTE = 0, 1, 2
DYMOE_ERR_CAPACITY = 7


class Pool:
    """dymoe_pool (include/dymoe.h): the mixed-precision expert pool's host-side policy."""

    def __init__(self, capacity):
        h = ctypes.c_void_p()
        _check(lib().dymoe_pool_create(capacity, ctypes.byref(h)))
        self.handle = h
        self.capacity = capacity

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.dymoe_pool_destroy(self.handle)
            self.handle = None

    def lookup(self, layer, expert, bits):
        out, served, off = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
        _check(lib().dymoe_pool_lookup(self.handle, layer, expert, bits, ctypes.byref(out),
                                       ctypes.byref(served), ctypes.byref(off)))
        return out.value, served.value, (off.value if out.value == POOL_HIT else None)

    def insert(self, layer, expert, bits, nbytes, max_evicted=256):
        off, n = ctypes.c_size_t(), ctypes.c_int()
        ev = (ctypes.c_int32 * (2 * max_evicted))()
        _check(lib().dymoe_pool_insert(self.handle, layer, expert, bits, nbytes, ctypes.byref(off),
                                       ev, max_evicted, ctypes.byref(n)))
        return off.value, [(ev[2 * i], ev[2 * i + 1]) for i in range(min(n.value, max_evicted))]

    def pin(self, layer, expert):
        _check(lib().dymoe_pool_pin(self.handle, layer, expert))

    def unpin(self, layer, expert):
        _check(lib().dymoe_pool_unpin(self.handle, layer, expert))

    def snapshot(self):
        n = ctypes.c_int()
        _check(lib().dymoe_pool_snapshot(self.handle, None, 0, ctypes.byref(n)))
        arr = (PoolEntry * max(n.value, 1))()
        _check(lib().dymoe_pool_snapshot(self.handle, arr, n.value, ctypes.byref(n)))
        return [((e.layer, e.expert), dict(bits=e.bits, nbytes=e.bytes, offset=e.offset,
                                           last_use=e.last_use, pins=e.pins)) for e in arr[:n.value]]

    def used(self):
        return lib().dymoe_pool_used(self.handle)


def make_opts(phase, layer, num_layers, ladder, attn_mass=None, k_tokens=0, ffn_mode=-1,
              out_dtype=DYMOE_OUT_F32, forced_bits=None, residual=None, prof_events=None):
    """dymoe_fwd_opts (include/dymoe.h) from tensors; prof_events: 3 torch.cuda.Events or None."""
    o = FwdOpts()
    o.phase = phase
    o.layer = layer
    o.num_layers = num_layers
    o.ladder = ladder
    o.attn_mass = _p(attn_mass)
    o.heads = attn_mass.shape[0] if attn_mass is not None else 0
    o.k_tokens = k_tokens
    o.ffn_mode = ffn_mode
    o.out_dtype = out_dtype
    o.forced_bits = _p(forced_bits)
    o.residual = _p(_u16(residual)) if residual is not None else None
    if prof_events is not None:
        for i, ev in enumerate(prof_events):
            o.prof_events[i] = ev.cuda_event
    return o


# ---------------------------------------------------------------------------------------------
class MoELayer:
    """An expert table (dymoe_layer handle).  `experts` is a list of dicts with bf16 masters
    'w1','w3' [F,Hd], 'w2' [Hd,F] (optional) and per quantized width b a dict 'q{b}' =
    {'w1': (codes, scales, zeros), 'w3': ..., 'w2': ...}.  Tensors must outlive the layer."""

    def __init__(self, experts, k_route, hidden, ffn):
        self.M = len(experts)
        self.k = k_route
        self.hidden = hidden
        self.ffn = ffn
        self._keep = list(experts)
        arr = (ExpertDesc * self.M)()
        for e, ex in enumerate(experts):
            _fill_desc(arr[e], ex)
        desc = LayerDesc(self.M, k_route, hidden, ffn, arr)
        h = ctypes.c_void_p()
        _check(lib().dymoe_layer_create(ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.dymoe_layer_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def set_expert(self, e, expert, stream=None):
        """dymoe_layer_set_expert: rebind expert e to the formats in `expert` (same dict layout
        as the constructor's; absent widths are unbound).  Stream-ordered."""
        d = ExpertDesc()
        _fill_desc(d, expert)
        _check(lib().dymoe_layer_set_expert(self.handle, e, ctypes.byref(d), _stream(stream)))
        self._keep[e] = expert

    def refresh(self, stream=None):
        """dymoe_layer_refresh: rebuild the derived dequant metadata after re-quantizing."""
        _check(lib().dymoe_layer_refresh(self.handle, _stream(stream)))

    def workspace(self, T, device="cuda"):
        n = lib().dymoe_workspace_size(self.handle, T)
        return torch.zeros(max(n, 256), dtype=torch.uint8, device=device)

    def views(self, T, ws):
        v = WsViews()
        _check(lib().dymoe_workspace_views(self.handle, T, _p(ws), ctypes.byref(v)))
        base = ws.data_ptr()
        M, k, Hd, F = self.M, self.k, self.hidden, self.ffn

        def view(name, shape, dtype):
            off = getattr(v, name) - base
            n = 1
            for s in shape:
                n *= s
            nbytes = n * torch.empty(0, dtype=dtype).element_size()
            return ws[off:off + nbytes].view(dtype).view(*shape)
        return dict(
            topk_idx=view("topk_idx", (T, k), torch.int32), topk_w=view("topk_w", (T, k), torch.float32),
            probs=view("probs", (T, M), torch.float32), importance=view("importance", (M,), torch.float32),
            heavy=view("heavy", (T,), torch.int32), bits=view("bits", (M,), torch.uint8),
            active=view("active", (M,), torch.uint8), expert_off=view("expert_off", (M + 1,), torch.int32),
            perm_token=view("perm_token", (T * k,), torch.int32), perm_slot=view("perm_slot", (T * k,), torch.int32),
            inv_row=view("inv_row", (T, k), torch.int32), h=view("h", (T * k, F), torch.bfloat16),
            y_perm=view("y_perm", (T * k, Hd), torch.float32), status=view("status", (1,), torch.int32))

    def ffn_workspace(self, T, device="cuda"):
        n = lib().dymoe_expert_ffn_ws_bytes(self.handle, T)
        return torch.empty(max(n, 256), dtype=torch.uint8, device=device)

    def expert_ffn_into(self, x_ptr, T, bits, expert_off, perm_token, mode, y_ptr, h, status,
                        ws=None, stream=None):
        """dymoe_expert_ffn on raw device rows (x_ptr [T][Hd] bf16) writing y_perm to y_ptr
        ([T*k][Hd] f32), e.g. an expert-parallel peer window; h [T*k][F] bf16 scratch."""
        ws = self.ffn_workspace(T, h.device) if ws is None else ws
        _check(lib().dymoe_expert_ffn(self.handle, mode, ctypes.c_void_p(x_ptr), T, _p(bits),
                                      _p(expert_off), _p(perm_token), _p(h), ctypes.c_void_p(y_ptr),
                                      _p(status), _p(ws), ws.numel(), _stream(stream)))

    def expert_ffn(self, x, bits, expert_off, perm_token, mode, ws=None, stream=None):
        T = x.shape[0]
        h = torch.empty(max(T * self.k, 1), self.ffn, dtype=torch.bfloat16, device=x.device)
        y = torch.empty(max(T * self.k, 1), self.hidden, dtype=torch.float32, device=x.device)
        status = torch.zeros(1, dtype=torch.int32, device=x.device)
        ws = self.ffn_workspace(T, x.device) if ws is None else ws
        _check(lib().dymoe_expert_ffn(self.handle, mode, _p(_u16(x)), T, _p(bits), _p(expert_off),
                                      _p(perm_token), _p(h), _p(y), _p(status), _p(ws), ws.numel(),
                                      _stream(stream)))
        return h, y, status

    def forward(self, x, logits, ladder, layer, num_layers, phase=DYMOE_DECODE, attn_mass=None,
                k_tokens=0, out_dtype=DYMOE_OUT_F32, forced_bits=None, ffn_mode=-1, ws=None,
                out=None, stream=None, prof_events=None, residual=None):
        """dymoe_moe_forward.  Returns (y, ws).  prof_events: optional 3 torch.cuda.Events
        (already recorded once so that they exist) recorded around the FFN kernels."""
        T = x.shape[0]
        if ws is None:
            ws = self.workspace(T, x.device)
        if out is None:
            out = torch.empty(T, self.hidden, device=x.device,
                              dtype=torch.float32 if out_dtype == DYMOE_OUT_F32 else torch.bfloat16)
        o = make_opts(phase, layer, num_layers, ladder, attn_mass, k_tokens, ffn_mode, out_dtype,
                      forced_bits, residual, prof_events)
        _check(lib().dymoe_moe_forward(self.handle, _p(_u16(x)), _p(logits), T, ctypes.byref(o),
                                       _p(out), _p(ws), ws.numel(), _stream(stream)))
        return out, ws

    def check_status(self, T, ws, stream=None):
        word = ctypes.c_uint32()
        rc = lib().dymoe_check_status(self.handle, T, _p(ws), ctypes.byref(word), _stream(stream))
        return rc, word.value


def quantize_experts(experts, widths=(8, 4, 2), stream=None):
    """Quantize every expert's W1/W3/W2 to each width in one batched launch (in place: adds
    'q{b}' entries)."""
    jobs = []
    for ex in experts:
        for b in widths:
            q = {}
            for n in ("w1", "w3", "w2"):
                W = ex[n]
                q[n] = alloc_qmat(W.shape[0], W.shape[1], b, W.device)
                jobs.append((W, b, q[n]))
            ex["q%d" % b] = q
    for i in range(0, len(jobs), 64):
        dymoe_quantize_batched(jobs[i:i + 64], stream=stream)
    return experts
