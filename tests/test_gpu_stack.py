"""GPU parity of the C5 layer stack (paper_2603_19172_b200.stack.MoEStack): 32 layers on the bf16
residual stream (pre-norm: RMSNorm -> router -> MoE -> residual add), each layer routed by its own
gate on the device, depth-adaptive bits.  Teacher-forced layer by layer against oracle.stack: the
GPU's normed input u_l is within one bf16 ulp of the oracle's RMSNorm of the GPU's x_l (fp32 vs
fp64 mean of squares; rare), and, fed the GPU's u_l, the oracle's exact router logits (reading P1)
must lie within the kernel's fp32 bound of the GPU's (tests/validity.py), the GPU's routing must be
a valid top-k under that bound (the oracle's wherever unambiguous), the bits the oracle's (decode
B > 1: a valid assignment under the gate-sum tolerance), and x_{l+1} within
|x_gpu - x_ref| <= 2e-3 max|y_ref| + ulp_bf16(x_ref) elementwise (the FFN bar of north_star plus one
rounding of the bf16 stream) on every token whose routing is unambiguous."""
import numpy as np
import pytest
import torch

import synthetic
from oracle import stack as o_stack, schedule as o_sched, moe as o_moe
from validity import check_bits, check_logits, check_topk, decode_importance_tol, gate_logit_bound

pytestmark = pytest.mark.gpu


def D():
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    return d


def _ulp_bf16(v):
    a = np.abs(v)
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    return np.where(a > 0, 2.0 ** (e - 7), 2.0 ** -133)


@pytest.mark.parametrize("phase,T", [("decode", 8), ("prefill", 40)])
def test_stack_32_layers_teacher_forced(phase, T):
    d = D()
    from paper_2603_19172_b200.stack import MoEStack
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    L = 32
    masters = [synthetic.expert_weights(cfg, 100 + l) for l in range(L)]
    gpu_layers = []
    for l in range(L):
        ex = [{n: t.cuda() for n, t in e.items()} for e in masters[l]]
        d.quantize_experts(ex, (8, 4, 2))
        gpu_layers.append(ex)
    gates = [synthetic.stack_gate(cfg, l, 5) for l in range(L)]
    st = MoEStack(gpu_layers, [(w.cuda(), b.cuda()) for w, b in gates], cfg.k, cfg.hidden, cfg.ffn)
    x0 = synthetic.hidden_states(cfg, 6).cuda()
    attn = [synthetic.attention_mass(cfg, 200 + l).cuda() for l in range(L)] if phase == "prefill" else None
    bits_t, lams = (8, 4, 2), (0.25, 0.5)
    ph = d.DYMOE_PREFILL if phase == "prefill" else d.DYMOE_DECODE
    xL, trace = st.forward(x0, d.make_ladder(bits_t, lams), phase=ph, attn_masses=attn, trace=True)
    torch.cuda.synchronize()
    lad = o_sched.Ladder(bits_t, lams)
    seen = set()
    n_u_diff = 0
    n_near = 0
    for l in range(L):
        x_in = trace[l][0].float().cpu().numpy()
        u_gpu = trace[l][1].float().cpu().numpy().astype(np.float64)
        u_ref = o_stack.rmsnorm(x_in)
        assert (np.abs(u_gpu - u_ref) <= _ulp_bf16(u_ref)).all(), "rmsnorm, layer %d" % l
        n_u_diff += int((u_gpu != u_ref).sum())
        x_out = (trace[l + 1][0] if l + 1 < L else xL).float().cpu().numpy().astype(np.float64)
        np_ex = [{n: t.float().numpy() for n, t in e.items()} for e in masters[l]]
        wg, beta = gates[l]
        x_ref, lg_ref, out = o_stack.stack_layer(
            x_in, wg.float().numpy(), beta.numpy(), np_ex, l, L, lad, cfg.k, phase=phase,
            attn_mass=attn[l].cpu().numpy() if attn is not None else None, u=u_gpu)
        bound = gate_logit_bound(u_gpu, wg.float().numpy(), lg_ref)
        check_logits(trace[l][2].cpu().numpy(), lg_ref, bound)
        idx_gpu = trace[l][4].cpu().numpy()
        near = check_topk(idx_gpu, lg_ref, bound)
        n_near += int(near.sum())
        bits = trace[l][3].cpu().numpy()
        tol = 0 if (phase == "prefill" or T == 1) else decode_importance_tol(T)
        if not near.any():
            assert np.array_equal(idx_gpu, out["topk_idx"]), "routing, layer %d" % l
            if not check_bits(bits, out["bits"], out["importance"], tol):
                # near-tied gate sums: the GPU's valid assignment; the FFN checked on its widths
                x_ref, _, out = o_stack.stack_layer(
                    x_in, wg.float().numpy(), beta.numpy(), np_ex, l, L, lad, cfg.k, phase=phase,
                    attn_mass=attn[l].cpu().numpy() if attn is not None else None, u=u_gpu,
                    forced_bits=bits)
        seen.update(int(b) for b in bits)
        ok = ~near if np.array_equal(bits, out["bits"]) else np.zeros(T, bool)
        bound = 2e-3 * np.abs(out["y"]).max() + _ulp_bf16(x_ref)
        assert (np.abs(x_out - x_ref) <= bound)[ok].all(), "stream, layer %d" % l
        assert ok.sum() >= T - 2
    assert n_near <= 2                 # ambiguous routings under the fp32 bound are rare
    assert np.isfinite(xL.float().cpu().numpy()).all()
    assert n_u_diff <= 0.01 * L * T * cfg.hidden          # 1-ulp norm differences are rare
    assert {8, 4, 2} <= seen          # the depth schedule used every tier along the stack


def test_rmsnorm_kernel():
    d = D()
    cfg = synthetic.CONFIGS["tiny"]
    x = (synthetic.hidden_states(cfg, 9).float() * 7.5).to(torch.bfloat16)
    u = d.dymoe_rmsnorm(x.cuda()).float().cpu().numpy().astype(np.float64)
    ref = o_stack.rmsnorm(x.float().numpy())
    assert (np.abs(u - ref) <= _ulp_bf16(ref)).all()
    assert (u != ref).mean() < 0.01
    with pytest.raises(d.DymoeError):
        xc = x.cuda()
        d.dymoe_rmsnorm(xc, out=xc)                                  # u aliases x


def test_gate_logits_bias_and_residual_args():
    d = D()
    cfg = synthetic.CONFIGS["tiny"]
    wg, beta = synthetic.stack_gate(cfg, 3, 1)
    x = synthetic.hidden_states(cfg, 2)
    lg = d.dymoe_gate_logits(x.cuda(), wg.cuda(), beta.cuda()).cpu().numpy()
    ref = o_stack.router_logits(x.float().numpy(), wg.float().numpy(), beta.numpy())
    check_logits(lg, ref, gate_logit_bound(x.float().numpy(), wg.float().numpy(), ref))
    lg0 = d.dymoe_gate_logits(x.cuda(), wg.cuda()).cpu().numpy()
    ref0 = o_stack.router_logits(x.float().numpy(), wg.float().numpy())
    check_logits(lg0, ref0, gate_logit_bound(x.float().numpy(), wg.float().numpy()))
    # the bias is one fp32 add of the kernel's own product (beta = 0 leaves it unchanged)
    assert np.array_equal(lg, (lg0 + beta.numpy()).astype(np.float32))
    with pytest.raises(d.DymoeError):
        d.dymoe_gate_logits(x.cuda()[:, :100].contiguous(), wg.cuda()[:, :100].contiguous())   # Hd % 8 != 0


@pytest.mark.parametrize("phase,T", [("decode", 8), ("prefill", 40)])
def test_ep_stack_single_rank_equals_stack(phase, T):
    """EPStack (one dymoe_ep handle serving every layer) on one rank, over the peer windows and
    over the library's NCCL communicator, gives MoEStack's stream bit for bit (same kernels, same
    arithmetic, one rank owning every expert)."""
    d = D()
    from paper_2603_19172_b200 import ep
    from paper_2603_19172_b200.stack import EPStack, MoEStack
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    L = 4
    layers = []
    for l in range(L):
        ex = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 140 + l)]
        d.quantize_experts(ex, (8, 4, 2))
        layers.append(ex)
    gates = [tuple(t.cuda() for t in synthetic.stack_gate(cfg, l, 4)) for l in range(L)]
    attn = [synthetic.attention_mass(cfg, 220 + l).cuda() for l in range(L)] if phase == "prefill" else None
    ph = d.DYMOE_PREFILL if phase == "prefill" else d.DYMOE_DECODE
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    x0 = synthetic.hidden_states(cfg, 7).cuda()
    ref, _ = MoEStack(layers, gates, cfg.k, cfg.hidden, cfg.ffn).forward(x0, lad, phase=ph, attn_masses=attn)
    h = ep.EPLayer(0, 1, cfg.M, cfg.k, cfg.hidden, cfg.ffn, T, layers[0],
                   transports=d.DYMOE_EP_NCCL | d.DYMOE_EP_PEER, nccl_uid=ep.unique_id())
    st = EPStack(h, layers, gates)
    for tp in (d.DYMOE_EP_PEER, d.DYMOE_EP_NCCL):
        y, _ = st.forward(x0, lad, phase=ph, transport=tp, attn_masses=attn)
        torch.cuda.synchronize()
        assert torch.equal(y, ref), tp
    h.close()


def test_ep_stack_two_ranks_teacher_forced():
    """EPStack over 2 ranks (threads, peer windows), 4 layers, decode: every layer of every rank
    against the oracle stack layer with the GLOBAL bits (both ranks' gate sums), teacher-forced."""
    import threading
    d = D()
    from paper_2603_19172_b200 import ep
    from paper_2603_19172_b200.stack import EPStack
    from oracle import importance as o_imp, route as o_route, moe as o_moe
    cfg = synthetic.CONFIGS["tiny"].with_tokens(8)
    L, P = 4, 2
    masters = [synthetic.expert_weights(cfg, 160 + l) for l in range(L)]
    layers = []
    for l in range(L):
        ex = [{n: t.cuda() for n, t in e.items()} for e in masters[l]]
        d.quantize_experts(ex, (8, 4, 2))
        layers.append(ex)
    gates = [synthetic.stack_gate(cfg, l, 4) for l in range(L)]
    gates_d = [tuple(t.cuda() for t in g) for g in gates]
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    hs, stacks = [], []
    for r in range(P):
        first, last = ep.owned_range(r, cfg.M, P)
        h = ep.EPLayer(r, P, cfg.M, cfg.k, cfg.hidden, cfg.ffn, cfg.T, layers[0][first:last])
        hs.append(h)
        stacks.append(EPStack(h, [lay[first:last] for lay in layers], gates_d))
    ep.connect_threads(hs)
    xs = [synthetic.hidden_states(cfg, 30 + r).cuda() for r in range(P)]
    wss = [h.workspace(cfg.T) for h in hs]
    bufs = [(torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)) for x in xs]
    lgs = [torch.empty(cfg.T, cfg.M, device="cuda") for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    torch.cuda.synchronize()
    res, errors = {}, []

    def worker(r):
        try:
            with torch.cuda.stream(streams[r]):
                y, tr = stacks[r].forward(xs[r], lad, d.DYMOE_DECODE, ws=wss[r], bufs=bufs[r],
                                          logits=lgs[r], trace=True)
                torch.cuda.current_stream().synchronize()
                res[r] = (y.float().cpu().numpy(), [tuple(t.cpu() for t in e) for e in tr])
        except Exception as e:   # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join() for t in th]
    [h.close() for h in hs]
    assert not errors, errors
    lad_o = o_sched.Ladder((8, 4, 2), (0.25, 0.5))
    np_ex = [[{n: t.float().numpy() for n, t in e.items()} for e in masters[l]] for l in range(L)]
    for l in range(L):
        wg, beta = gates[l]
        I = np.zeros(cfg.M)
        lg_ref = {}
        for r in range(P):
            u = res[r][1][l][1].float().numpy().astype(np.float64)
            lg_ref[r] = o_stack.router_logits(u, wg.float().numpy(), beta.numpy())
            _, _, p = o_route.route(lg_ref[r], cfg.k)
            I = I + o_imp.decode_importance(lg_ref[r], p)
        bits_ref, _ = o_sched.assign_bits(I, l, L, lad_o, cfg.k)
        for r in range(P):
            x_in, u, _, bits, idx = res[r][1][l]
            assert np.array_equal(bits.numpy(), res[0][1][l][3].numpy())
            check_bits(bits.numpy(), bits_ref, I, decode_importance_tol(cfg.T * P))
            assert np.array_equal(idx.numpy(), o_route.route(lg_ref[r], cfg.k)[0])
            y_ref = o_moe.moe_forward(u.float().numpy(), lg_ref[r], np_ex[l], l, L, lad_o, cfg.k,
                                      forced_bits=bits.numpy())["y"]
            xin = x_in.float().numpy().astype(np.float64)
            full = o_stack.residual(xin, y_ref)
            x_out = (res[r][1][l + 1][0].float().numpy() if l + 1 < L else res[r][0]).astype(np.float64)
            bound = 2e-3 * np.abs(y_ref).max() + _ulp_bf16(full)
            assert (np.abs(x_out - full) <= bound).all(), (r, l)
