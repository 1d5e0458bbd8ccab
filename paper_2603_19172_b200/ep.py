"""Expert-parallel DyMoE layer: a thin binding of the C ABI's dymoe_ep handle (include/dymoe.h
"The expert-parallel layer"; BASELINE.json north_star: "expert-parallel partitioning across 2, 4
and 8 GPUs ... NCCL all-to-all over NVLink for token dispatch and combine").

Everything of the step runs inside libdymoe: routing and scoring of the local tokens, the global
importance (sum over ranks), the bit assignment, the permutation, the exchange of the routed rows
(the handle's own NCCL communicator, or the peer-memory windows with fused dispatch / combine
kernels and device flag barriers), the owners' fused-dequant FFN and the weighted combine.  This
module only marshals arguments: the NCCL unique id travels from rank 0 over the caller's
torch.distributed group, window bases between threads of one process go through a Python list,
and between processes (CUDA IPC handles) through the process group.

Experts live on rank floor(e P / M) (contiguous blocks, `owned_range`), the same formula the
library uses.
"""
import ctypes

import torch

from . import dymoe as d


def owner_of(e, M, P):
    return (e * P) // M


def owned_range(rank, M, P):
    """[first, last) experts owned by `rank` (contiguous blocks, floor(e*P/M) == rank)."""
    first = -(-rank * M // P)
    last = -(-(rank + 1) * M // P)
    return first, last


def unique_id():
    """A fresh NCCL unique id (bytes) -- call on rank 0 and broadcast."""
    buf = ctypes.create_string_buffer(d.EP_UID_BYTES)
    d._check(d.lib().dymoe_ep_unique_id(buf))
    return bytes(buf.raw)


def broadcast_unique_id(group=None):
    """rank 0's NCCL unique id on every rank of a torch.distributed group (plumbing only)."""
    import torch.distributed as dist
    obj = [unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                               group=group)
    return obj[0]


class EPLayer:
    """One rank's share of an expert-parallel layer.

    local_experts: the expert dicts (bf16 masters + 'q{b}' packed widths, see dymoe.MoELayer) of
    the experts this rank owns, in order.  transports: mask of dymoe.DYMOE_EP_NCCL /
    DYMOE_EP_PEER.  nccl_uid: bytes from `unique_id()` on rank 0 (required for NCCL; with PEER it
    also lets the handle exchange the windows itself).  Without it, PEER windows are connected by
    the caller: `connect([base of every rank])`."""

    def __init__(self, rank, world, M, k, hidden, ffn, max_tokens, local_experts,
                 transports=d.DYMOE_EP_PEER, nccl_uid=None):
        self.rank, self.world = rank, world
        self.M, self.k, self.hidden, self.ffn = M, k, hidden, ffn
        self.first, self.last = owned_range(rank, M, world)
        assert len(local_experts) == self.last - self.first
        self.local = d.MoELayer(local_experts, 1, hidden, ffn)
        cfg = d.EpConfig(M, k, hidden, ffn, max_tokens, transports)
        h = ctypes.c_void_p()
        uid = ctypes.create_string_buffer(bytes(nccl_uid), d.EP_UID_BYTES) if nccl_uid else None
        d._check(d.lib().dymoe_ep_create(rank, world, uid, ctypes.byref(cfg), ctypes.byref(h)))
        self.handle = h

    def window(self):
        """(base pointer, 64-byte CUDA IPC handle) of this rank's window."""
        base = ctypes.c_void_p()
        ipc = ctypes.create_string_buffer(d.EP_IPC_BYTES)
        d._check(d.lib().dymoe_ep_window_base(self.handle, ctypes.byref(base), ipc))
        return base.value, bytes(ipc.raw)

    def connect(self, bases):
        arr = (ctypes.c_void_p * self.world)(*bases)
        d._check(d.lib().dymoe_ep_connect(self.handle, arr))

    def workspace(self, T, T_peer_max=0, placement=d.DYMOE_EP_ALL_TO_ALL, device="cuda"):
        n = d.lib().dymoe_ep_workspace_size(self.handle, T, T_peer_max, placement)
        return torch.zeros(max(n, 256), dtype=torch.uint8, device=device)

    def forward(self, x, logits, ladder, layer, num_layers, phase, transport=d.DYMOE_EP_PEER,
                placement=d.DYMOE_EP_ALL_TO_ALL, attn_mass=None, k_tokens=0, T_peer_max=0,
                out_dtype=d.DYMOE_OUT_F32, forced_bits=None, ffn_mode=-1, residual=None,
                prof_events=None, ws=None, out=None, stream=None, local=None):
        """dymoe_moe_forward_ep.  Returns (y, ws).  local: another dymoe.MoELayer of this rank's
        experts (same shapes) to run instead of the one given at construction -- one handle (one
        window) serves every layer of a stack."""
        local = self.local if local is None else local
        T = x.shape[0]
        if ws is None:
            ws = self.workspace(T, T_peer_max, placement, x.device)
        if out is None:
            out = torch.empty(T, self.hidden, device=x.device,
                              dtype=torch.float32 if out_dtype == d.DYMOE_OUT_F32 else torch.bfloat16)
        o = d.make_opts(phase, layer, num_layers, ladder, attn_mass, k_tokens, ffn_mode, out_dtype,
                        forced_bits, residual, prof_events)
        d._check(d.lib().dymoe_moe_forward_ep(
            self.handle, local.handle, transport, placement, d._p(d._u16(x)), d._p(logits), T,
            T_peer_max, ctypes.byref(o), d._p(out) if T else None, d._p(ws), ws.numel(),
            d._stream(stream)))
        return out, ws

    def views(self, T, ws, T_peer_max=0, placement=d.DYMOE_EP_ALL_TO_ALL):
        v = d.WsViews()
        d._check(d.lib().dymoe_ep_workspace_views(self.handle, T, T_peer_max, placement, d._p(ws),
                                                  ctypes.byref(v)))
        base, M, k = ws.data_ptr(), self.M, self.k

        def view(name, shape, dtype):
            off = getattr(v, name) - base
            n = 1
            for s in shape:
                n *= s
            nbytes = n * torch.empty(0, dtype=dtype).element_size()
            return ws[off:off + nbytes].view(dtype).view(*shape)
        return dict(
            topk_idx=view("topk_idx", (T, k), torch.int32), topk_w=view("topk_w", (T, k), torch.float32),
            importance=view("importance", (M,), torch.float32), bits=view("bits", (M,), torch.uint8),
            expert_off=view("expert_off", (M + 1,), torch.int32),
            inv_row=view("inv_row", (T, k), torch.int32), status=view("status", (1,), torch.int32))

    def check_status(self, T, ws, T_peer_max=0, placement=d.DYMOE_EP_ALL_TO_ALL, stream=None):
        word = ctypes.c_uint32()
        rc = d.lib().dymoe_ep_check_status(self.handle, T, T_peer_max, placement, d._p(ws),
                                           ctypes.byref(word), d._stream(stream))
        return rc, word.value

    def close(self):
        if getattr(self, "handle", None) is not None and d._lib is not None:
            d._check(d._lib.dymoe_ep_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def connect_threads(layers):
    """Connect the windows of P EPLayers that are threads of one process (same pointers)."""
    bases = [l.window()[0] for l in layers]
    for l in layers:
        l.connect(bases)


def connect_processes(layer, group=None):
    """Connect this process's window with its peers' over a torch.distributed group (CUDA IPC
    handles all-gathered and opened); returns the opened bases (closed by `disconnect`)."""
    import torch.distributed as dist
    base, ipc = layer.window()
    handles = [None] * layer.world
    dist.all_gather_object(handles, ipc, group=group)
    bases, opened = [], []
    for r, h in enumerate(handles):
        if r == layer.rank:
            bases.append(base)
        else:
            b = d.dymoe_ep_window_open(h)
            opened.append(b)
            bases.append(b)
    layer.connect(bases)
    return opened


def disconnect(opened):
    for b in opened:
        d.dymoe_ep_window_close(b)
