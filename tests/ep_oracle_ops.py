"""CPU stand-ins for the EP layer primitives, backed by the oracle (test infrastructure only).

They let the multi-process gloo tests exercise the expert-parallel orchestration of
paper_2603_19172_b200.ep (counts, splits, all-to-all order, local regrouping, reverse exchange,
combine) on CPU, where the CUDA kernels cannot run.  Every primitive here is the oracle's
definition of the corresponding C-ABI call.
"""
import numpy as np
import torch

from oracle import route as o_route, importance as o_imp, schedule as o_sched, moe as o_moe


def _ladder(ctypes_ladder):
    n = ctypes_ladder.n_tiers
    return o_sched.Ladder(bits=tuple(ctypes_ladder.bits[i] for i in range(n)),
                          lambdas=tuple(ctypes_ladder.lambdas[i] for i in range(n - 1)),
                          clamp_to_k=bool(ctypes_ladder.clamp_to_k),
                          m_active=bool(ctypes_ladder.m_mode),
                          renorm_on_skip=bool(ctypes_ladder.renorm_on_skip))


class SimpleLadder:
    """Duck-typed stand-in for the ctypes dymoe_ladder (no library needed on CPU)."""

    def __init__(self, bits, lambdas, clamp_to_k=True, m_active=False, renorm=True):
        self.n_tiers = len(bits)
        self.bits = list(bits) + [0] * (5 - len(bits))
        self.lambdas = list(lambdas) + [0.0] * (4 - len(lambdas))
        self.clamp_to_k = int(clamp_to_k)
        self.m_mode = int(m_active)
        self.renorm_on_skip = int(renorm)


class OracleOps:
    y_dtype = torch.float64

    def route(self, logits, k):
        idx, w, p = o_route.route(logits.numpy(), k)
        return torch.from_numpy(idx), torch.from_numpy(w), torch.from_numpy(p)

    def score(self, phase, M, k, topk_idx, attn_mass, logits, k_tokens):
        if phase == 0:
            I, _, _ = o_imp.score_prefill(attn_mass.numpy(), topk_idx.numpy(), M, k_tokens or None)
            return torch.from_numpy(I.astype(np.float64))
        _, _, p = o_route.route(logits.numpy(), 1)
        return torch.from_numpy(o_imp.decode_importance(logits.numpy(), p))

    def assign_bits(self, importance, layer, num_layers, ladder, k_route):
        bits, _ = o_sched.assign_bits(importance.numpy(), layer, num_layers, _ladder(ladder), k_route)
        return torch.from_numpy(bits)

    def permute(self, topk_idx, M, bits):
        r = o_moe.permute(topk_idx.numpy(), bits.numpy(), M)
        return (torch.from_numpy(r["expert_off"]), torch.from_numpy(r["perm_token"]),
                torch.from_numpy(r["perm_slot"]), torch.from_numpy(r["inv_row"]))

    def ep_plan(self, expert_off, P):
        off = expert_off.numpy()
        M = len(off) - 1
        counts = np.zeros(P, np.int32)
        rows = []
        for e in range(M):
            n = int(off[e + 1] - off[e])
            counts[(e * P) // M] += n
            rows += [e] * n
        return torch.from_numpy(counts), torch.tensor(rows, dtype=torch.int32)

    def gather_rows(self, x, rows):
        return x[rows.long()]

    def expert_ffn(self, layer, x_rows, bits, expert_off, perm_token, mode):
        # layer: list of numpy expert dicts of this rank's experts
        off = expert_off.numpy()
        y = np.zeros((max(int(off[-1]), 1), x_rows.shape[1]))
        for e in range(len(off) - 1):
            lo, hi = int(off[e]), int(off[e + 1])
            if hi == lo:
                continue
            W1, W3, W2 = o_moe.expert_weights(layer[e], int(bits[e]))
            xr = x_rows.numpy()[perm_token.numpy()[lo:hi]].astype(np.float64)
            y[lo:hi] = o_moe.ffn(xr, W1, W3, W2)
        return torch.from_numpy(y)

    def combine(self, y_rows, inv_row, weights, renorm):
        return torch.from_numpy(o_moe.combine(y_rows.numpy().astype(np.float64), inv_row.numpy(),
                                              weights.numpy().astype(np.float64), renorm))

    def renorm_weights(self, topk_idx, topk_w, bits, renorm):
        idx, w, b = topk_idx.numpy(), topk_w.numpy().astype(np.float64), bits.numpy()
        out = np.zeros_like(w)
        for t in range(idx.shape[0]):
            live = [s for s in range(idx.shape[1]) if b[idx[t, s]] > 0]
            den = sum(w[t, s] for s in live) if renorm else 1.0
            for s in live:
                out[t, s] = w[t, s] / den
        return torch.from_numpy(out)
