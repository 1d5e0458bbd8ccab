"""Expert-parallel DyMoE layer (BASELINE.json north_star: "expert-parallel partitioning across
2, 4 and 8 GPUs ... with an NCCL all-to-all over NVLink for token dispatch and combine";
SURVEY §8e).

Experts are sharded in contiguous blocks: expert e lives on rank floor(e * P / M).  One layer
step on every rank (each rank owns its own tokens -- weak scaling):

  1. route the local tokens (dymoe_route) and score them (dymoe_score);
  2. make the importance global: all-reduce(sum) of the per-rank importance vectors (exact
     integer counts in prefill; fp32 gate sums in decode).  Every rank receives the identical
     vector, so every rank computes the identical bit assignment (dymoe_assign_bits);
  3. permute the (token, slot) pairs by expert (dymoe_permute) -- because the owner is
     non-decreasing in e this order is already (destination rank, expert, token, slot);
     skipped experts' pairs are dropped and never sent; dymoe_ep_plan gives the per-destination
     row counts and the expert of every row;
  4. exchange counts, then all-to-all the gathered bf16 token rows (dymoe_gather_rows) and their
     expert ids;
  5. on the receiving rank: group the received rows by local expert (dymoe_permute with k = 1),
     run the fused-dequant expert FFN on its own experts (dymoe_expert_ffn) and put the fp32
     outputs back into received order (dymoe_combine with unit weights: exact);
  6. reverse all-to-all of the fp32 rows, and the weighted combine at the source
     (dymoe_combine with the routing weights).

Decode variant with the batch REPLICATED on every rank (decode at B <= 8 is latency
bound; `forward_replicated`): every rank routes, scores and assigns the same batch (identical
results, no exchange), runs only its own experts on the pairs routed to them, combines those
terms with weights renormalised over the GLOBAL live set (dymoe_renorm_weights, D12), and one
all-reduce(sum) of y [B][Hd] fp32 adds the ranks' partial outputs.  With top-2 each element has at
most two nonzero terms, so the sum does not depend on the reduction order.

Peer-memory variant (`forward_p2p`, SURVEY §8e over NVLink / NVSwitch): the two all-to-alls are
replaced by libdymoe kernels that move the rows themselves through symmetric windows mapped into
every rank (PeerWindows; CUDA IPC between processes): dymoe_ep_dispatch gathers each permuted row
and stores it straight into its owner's window at its final expert-major row (no regrouping on the
receiver), the FFN writes its outputs into the own window, and dymoe_ep_combine pulls every live
slot's output row from its owner and applies the weighted combine in the same kernel.  Three
flag barriers per step (dymoe_ep_barrier); the receive count is read once on the host to size
the FFN launch.

Every step of the math runs in libdymoe kernels; torch.distributed (NCCL on GPUs) carries the
bytes.  The only host synchronisation is the count exchange needed to size the all-to-all.
The orchestration is written against two small interfaces -- `ops` (the layer primitives) and
`comm` (the collectives) -- so that the same code runs with the CUDA ops over NCCL in
production, and is checked on CPU by the gloo multi-process tests with oracle-backed ops.
"""
import threading

import torch


def owner_of(e, M, P):
    return (e * P) // M


def owned_range(rank, M, P):
    """[first, last) experts owned by `rank` (contiguous blocks, floor(e*P/M) == rank)."""
    first = -(-rank * M // P)
    last = -(-(rank + 1) * M // P)
    return first, last


class TorchComm:
    """Collectives over a torch.distributed process group (NCCL between GPUs).  stage_cpu: move
    the payloads through host memory (gloo process groups, e.g. several test ranks sharing one
    GPU); never used for reported numbers."""

    def __init__(self, group=None, stage_cpu=False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.stage = stage_cpu

    def all_reduce_sum(self, t):
        if self.stage and t.is_cuda:
            c = t.cpu()
            self.dist.all_reduce(c, op=self.dist.ReduceOp.SUM, group=self.group)
            t.copy_(c)
            return t
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def exchange_counts(self, send_counts):
        src = send_counts.cpu() if self.stage else send_counts
        recv = torch.empty_like(src)
        self.dist.all_to_all_single(recv, src, group=self.group)
        return recv.to(send_counts.device)

    def all_to_all(self, send, send_splits, recv_splits):
        src = send.contiguous().cpu() if self.stage else send.contiguous()
        out = torch.empty((sum(recv_splits),) + tuple(send.shape[1:]), dtype=send.dtype,
                          device=src.device)
        self.dist.all_to_all_single(out, src, recv_splits, send_splits, group=self.group)
        return out.to(send.device)


class ThreadComm:
    """P ranks simulated by P threads of one process on one device (tests / single-GPU runs of
    the multi-rank path).  Collectives copy through shared slots behind a barrier."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.local = threading.local()

    def bind(self, rank):
        self.local.rank = rank
        return self

    @property
    def rank(self):
        return self.local.rank

    def _exchange(self, obj):
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.barrier.wait()
        self.slots[self.rank] = obj
        self.barrier.wait()
        got = list(self.slots)
        self.barrier.wait()
        return got

    def all_reduce_sum(self, t):
        parts = self._exchange(t.clone())
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p.to(acc.device)   # rank order: identical result on every rank
        t.copy_(acc)
        return t

    def exchange_counts(self, send_counts):
        parts = self._exchange(send_counts.clone())
        return torch.stack([p[self.rank] for p in parts]).to(send_counts.device)

    def all_to_all(self, send, send_splits, recv_splits):
        parts = self._exchange((send.clone(), list(send_splits)))
        chunks = []
        for src, (buf, splits) in enumerate(parts):
            start = sum(splits[: self.rank])
            chunks.append(buf[start:start + splits[self.rank]].to(send.device))
        out = torch.cat(chunks) if chunks else send[:0]
        assert out.shape[0] == sum(recv_splits)
        return out


class PeerWindows:
    """This rank's symmetric expert-parallel window and every peer's, mapped into this process
    (include/dymoe.h "Expert-parallel dispatch and combine over peer memory").

    comm: ThreadComm (ranks are threads of one process: the base pointers are shared directly) or
    TorchComm (one process per rank: 64-byte CUDA IPC handles are all-gathered and opened).
    barrier: "device" -- flag barriers in the windows (dymoe_ep_barrier, no host involvement);
    "host" -- stream synchronise + process-group barrier (ranks time-sharing ONE GPU from several
    processes, where a spinning device barrier would wait on context switches)."""

    def __init__(self, comm, M, hidden, cap_rows, barrier="device", device=None):
        from . import dymoe as d
        self.d, self.comm = d, comm
        self.P, self.rank = comm.world, comm.rank
        self.M, self.hidden, self.cap = M, hidden, cap_rows
        self.barrier_mode = barrier
        self.nbytes = d.dymoe_ep_window_bytes(self.P, M, hidden, cap_rows)
        self.base, handle = d.dymoe_ep_window_alloc(self.nbytes)
        self.opened = []
        if isinstance(comm, ThreadComm):
            bases = comm._exchange(self.base)
        else:
            handles = [None] * self.P
            comm.dist.all_gather_object(handles, handle, group=comm.group)
            bases = []
            for r, h in enumerate(handles):
                if r == self.rank:
                    bases.append(self.base)
                else:
                    b = d.dymoe_ep_window_open(h)
                    self.opened.append(b)
                    bases.append(b)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.peers = torch.tensor(bases, dtype=torch.int64, device=dev)
        self.win = d.EpWindow(self.P, self.rank, M, hidden, cap_rows, 0, self.peers.data_ptr())
        # the window's sections (include/dymoe.h): flags, cnt[2][P][M], recv_x, y_out
        a = lambda v: (v + 255) // 256 * 256
        cnt = a(self.P * 4)
        self.recv_x_ptr = self.base + cnt + a(2 * self.P * M * 4)
        self.y_out_ptr = self.recv_x_ptr + a(cap_rows * hidden * 2)
        self.epoch = 0
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ident = torch.arange(max(cap_rows, 1), dtype=torch.int32, device=dev)

    def barrier(self):
        if self.barrier_mode == "host":
            torch.cuda.current_stream().synchronize()
            if isinstance(self.comm, ThreadComm):
                self.comm.barrier.wait()
            else:
                self.comm.dist.barrier(group=self.comm.group)
            return
        self.epoch += 1
        self.d.dymoe_ep_barrier(self.win, self.epoch, self.status)

    def close(self):
        for b in self.opened:
            self.d.dymoe_ep_window_close(b)
        self.opened = []
        if self.base:
            torch.cuda.synchronize()
            self.d.dymoe_ep_window_free(self.base)
            self.base = None


class CudaOps:
    """The layer primitives on the CUDA path (libdymoe C ABI)."""

    y_dtype = torch.float32

    def __init__(self):
        from . import dymoe as d
        d.lib()
        self.d = d

    def route(self, logits, k):
        return self.d.dymoe_route(logits, k)

    def score(self, phase, M, k, topk_idx, attn_mass, logits, k_tokens):
        imp, _ = self.d.dymoe_score(phase, M, k, topk_idx=topk_idx, attn_mass=attn_mass,
                                    logits=logits, k_tokens=k_tokens)
        return imp

    def assign_bits(self, importance, layer, num_layers, ladder, k_route):
        return self.d.dymoe_assign_bits(importance, layer, num_layers, ladder, k_route)[0]

    def permute(self, topk_idx, M, bits):
        return self.d.dymoe_permute(topk_idx, M, bits)

    def ep_plan(self, expert_off, P):
        return self.d.dymoe_ep_plan(expert_off, P)

    def gather_rows(self, x, rows):
        return self.d.dymoe_gather_rows(x, rows)

    def expert_ffn(self, layer, x_rows, bits, expert_off, perm_token, mode):
        return layer.expert_ffn(x_rows, bits, expert_off, perm_token, mode)[1]

    def combine(self, y_rows, inv_row, weights, renorm):
        return self.d.dymoe_combine(y_rows, inv_row, weights, renorm=renorm)

    def renorm_weights(self, topk_idx, topk_w, bits, renorm):
        return self.d.dymoe_renorm_weights(topk_idx, topk_w, bits, renorm=renorm)


class EPMoELayer:
    """One rank's shard of an expert-parallel DyMoE layer.

    local_experts: the expert dicts (bf16 masters + 'q{b}' packed widths, see MoELayer) of the
    experts this rank owns, in order; `make_local_layer(experts)` builds the local expert table
    (a dymoe.MoELayer with k_route = 1 on the CUDA path)."""

    def __init__(self, comm, ops, local_experts, M, k, hidden, ffn, make_local_layer):
        self.comm, self.ops = comm, ops
        self.M, self.k, self.hidden, self.ffn = M, k, hidden, ffn
        self.P = comm.world
        self.first, self.last = owned_range(comm.rank, M, self.P)
        assert len(local_experts) == self.last - self.first
        self.local = make_local_layer(local_experts) if local_experts else None

    def forward(self, x, logits, ladder, layer, num_layers, phase, attn_mass=None, k_tokens=0,
                renorm=True, ffn_mode=None):
        ops, comm = self.ops, self.comm
        M, k, P = self.M, self.k, self.P
        PREFILL, DECODE = 0, 1
        T = x.shape[0]
        idx, w, probs = ops.route(logits, k)
        # 2. global importance (identical on every rank after the all-reduce)
        if phase == DECODE and P > 1 and T == 1:
            imp = probs[0].clone()          # g of the single local token (Eq. 3)
        else:
            imp = ops.score(phase, M, k, idx, attn_mass, logits, k_tokens)
        if P > 1:
            imp = comm.all_reduce_sum(imp)   # prefill: exact counts; decode: sum of gates
        bits = ops.assign_bits(imp, layer, num_layers, ladder, k)
        # 3. permutation (destination-rank ordered) and the send plan
        off, pt, ps, inv = ops.permute(idx, M, bits)
        send_counts, row_expert = ops.ep_plan(off, P)
        R = int(off[-1].item())
        # 4. counts, then rows + their expert ids (the one host synchronisation)
        recv_counts = comm.exchange_counts(send_counts)
        send_splits = [int(v) for v in send_counts.tolist()]
        recv_splits = [int(v) for v in recv_counts.tolist()]
        x_send = ops.gather_rows(x, pt[:R])
        x_recv = comm.all_to_all(x_send, send_splits, recv_splits)
        e_recv = comm.all_to_all(row_expert[:R], send_splits, recv_splits)
        n_recv = x_recv.shape[0]
        # 5. local experts on the received rows
        if n_recv > 0:
            M_loc = self.last - self.first
            loc_idx = (e_recv - self.first).to(torch.int32).reshape(n_recv, 1).contiguous()
            bits_loc = bits[self.first:self.last].contiguous()
            off_l, pt_l, _, inv_l = ops.permute(loc_idx, M_loc, bits_loc)
            mode = (PREFILL if n_recv > 64 else DECODE) if ffn_mode is None else ffn_mode
            y_loc = ops.expert_ffn(self.local, x_recv, bits_loc, off_l, pt_l, mode)
            ones = torch.ones(n_recv, 1, dtype=torch.float32, device=x.device)   # exact reorder
            y_recv = ops.combine(y_loc, inv_l, ones, False)
        else:
            y_recv = torch.zeros(0, self.hidden, dtype=ops.y_dtype, device=x.device)
        # 6. back to the sources, weighted combine
        y_back = comm.all_to_all(y_recv, recv_splits, send_splits)
        if y_back.shape[0] == 0:
            y_back = torch.zeros(1, self.hidden, dtype=ops.y_dtype, device=x.device)
        y = ops.combine(y_back, inv, w, renorm)
        return y, dict(bits=bits, importance=imp, topk_idx=idx, topk_w=w, send=send_splits,
                       recv=recv_splits)

    def forward_p2p(self, win, x, logits, ladder, layer, num_layers, phase, attn_mass=None,
                    k_tokens=0, renorm=True, ffn_mode=None):
        """forward() with dispatch and combine over peer memory (`win`: PeerWindows).  Same
        result as forward(), bit for bit: the receive layout is the expert-major order forward()
        regroups into, and the combine is dymoe_combine's arithmetic."""
        ops, comm, d = self.ops, self.comm, win.d
        M, k, P = self.M, self.k, self.P
        PREFILL, DECODE = 0, 1
        idx, w, probs = ops.route(logits, k)
        if phase == DECODE and P > 1 and x.shape[0] == 1:
            imp = probs[0].clone()
        else:
            imp = ops.score(phase, M, k, idx, attn_mass, logits, k_tokens)
        if P > 1:
            imp = comm.all_reduce_sum(imp)
        bits = ops.assign_bits(imp, layer, num_layers, ladder, k)
        off, pt, ps, inv = ops.permute(idx, M, bits)
        # counts into every window, then the rows straight to their owners
        d.dymoe_ep_publish_counts(win.win, off)
        win.barrier()
        M_loc = self.last - self.first
        recv_off = torch.empty(M_loc + 1, dtype=torch.int32, device=x.device)
        d.dymoe_ep_dispatch(win.win, x, off, pt, recv_off, win.status)
        win.barrier()
        n_recv = int(recv_off[M_loc].item())      # sizes the FFN launch (one host read)
        if n_recv > 0:
            mode = (PREFILL if n_recv > 64 else DECODE) if ffn_mode is None else ffn_mode
            bits_loc = bits[self.first:self.last].contiguous()
            h = torch.empty(n_recv, self.ffn, dtype=torch.bfloat16, device=x.device)
            self.local.expert_ffn_into(win.recv_x_ptr, n_recv, bits_loc, recv_off,
                                       win.ident[:n_recv], mode, win.y_out_ptr, h, win.status)
        win.barrier()
        y = d.dymoe_ep_combine(win.win, inv, w, off, renorm=renorm)
        win.win.parity ^= 1
        return y, dict(bits=bits, importance=imp, topk_idx=idx, topk_w=w, recv=n_recv)

    def forward_replicated(self, x, logits, ladder, layer, num_layers, k_tokens=0, renorm=True,
                           ffn_mode=None):
        """Decode with the same batch x [B][Hd] on every rank (see the module docstring).
        Returns (y [B][Hd] summed over the ranks, info)."""
        ops, comm = self.ops, self.comm
        M, k = self.M, self.k
        DECODE = 1
        B = x.shape[0]
        idx, w, probs = ops.route(logits, k)
        imp = ops.score(DECODE, M, k, idx, None, logits, k_tokens)
        bits = ops.assign_bits(imp, layer, num_layers, ladder, k)
        wn = ops.renorm_weights(idx, w, bits, renorm)
        # local view: this rank's experts keep their index (shifted) and width; every other
        # expert maps to one extra skipped slot M_loc, so its pairs are dropped by the permute
        M_loc = self.last - self.first
        mine = (idx >= self.first) & (idx < self.last)
        idx_loc = torch.where(mine, idx - self.first, torch.full_like(idx, M_loc)).contiguous()
        bits_loc = torch.cat([bits[self.first:self.last], bits.new_zeros(1)]).contiguous()
        off, pt, _, inv = ops.permute(idx_loc, M_loc + 1, bits_loc)
        n_rows = int(off[M_loc].item()) if M_loc > 0 else 0
        if n_rows > 0:
            # the local table is a k = 1 layer: hand it the routed rows themselves (expert order)
            mode = DECODE if ffn_mode is None else ffn_mode
            x_rows = ops.gather_rows(x, pt[:n_rows].contiguous())
            ident = torch.arange(n_rows, dtype=torch.int32, device=x.device)
            y_loc = ops.expert_ffn(self.local, x_rows, bits_loc[:M_loc].contiguous(),
                                   off[:M_loc + 1].contiguous(), ident, mode)
        else:
            y_loc = torch.zeros(1, self.hidden, dtype=ops.y_dtype, device=x.device)
        y = ops.combine(y_loc, inv, wn, False)
        if self.P > 1:
            y = comm.all_reduce_sum(y)
        return y, dict(bits=bits, importance=imp, topk_idx=idx, topk_w=w, rows=n_rows)
