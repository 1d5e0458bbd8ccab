import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synthetic
import paper_2603_19172_b200.dymoe as d
from paper_2603_19172_b200.stack import MoEStack
cfg = synthetic.CONFIGS["tiny"].with_tokens(8)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
layers = []
for l in range(L):
    ex = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 100 + l)]
    d.quantize_experts(ex, (8, 4, 2))
    layers.append(ex)
gates = [tuple(t.cuda() for t in synthetic.stack_gate(cfg, l, 5)) for l in range(L)]
x = synthetic.hidden_states(cfg, 6).cuda()
lg = d.dymoe_gate_logits(x, gates[0][0], gates[0][1]); torch.cuda.synchronize(); print("gate ok", lg[0])
L0 = d.MoELayer(layers[0], cfg.k, cfg.hidden, cfg.ffn)
y, ws = L0.forward(x, lg, d.make_ladder((8, 4, 2), (0.25, 0.5)), 0, 32); torch.cuda.synchronize(); print("fwd f32 ok")
yb = torch.empty_like(x)
y, ws = L0.forward(x, lg, d.make_ladder((8, 4, 2), (0.25, 0.5)), 0, 32, out=yb, out_dtype=d.DYMOE_OUT_BF16); torch.cuda.synchronize(); print("fwd bf16 ok")
y, ws = L0.forward(x, lg, d.make_ladder((8, 4, 2), (0.25, 0.5)), 0, 32, out=yb, out_dtype=d.DYMOE_OUT_BF16, residual=x); torch.cuda.synchronize(); print("fwd residual ok")
st = MoEStack(layers, gates, cfg.k, cfg.hidden, cfg.ffn)
cur = x
for l in range(L):
    y, _ = st.forward(cur, d.make_ladder((8, 4, 2), (0.25, 0.5)), first_layer=l, n_layers=1)
    torch.cuda.synchronize()
    lg = d.dymoe_gate_logits(cur, gates[l][0], gates[l][1])
    print(l, "x max", cur.float().abs().max().item(), "finite", bool(torch.isfinite(cur.float()).all()),
          "logits max", lg.abs().max().item(), "y max", y.float().abs().max().item(), flush=True)
    cur = y.clone()
