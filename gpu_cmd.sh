timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -5
python - <<'PY'
import torch
import paper_2603_19172_b200.dymoe as d
d.lib()
H, T = 32, 2048
q = torch.randn(H, T, 128, device='cuda').to(torch.bfloat16)
k = torch.randn(H, T, 128, device='cuda').to(torch.bfloat16)
for _ in range(3): d.dymoe_attention_mass(q, k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): d.dymoe_attention_mass(q, k)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
fl = 2 * 2 * T * T * 128 * H / 2
print('attention mass H=32 T=2048: %.1f us, %.0f TFLOP/s (two causal QK^T passes)' % (ms * 1e3, fl / ms / 1e9))
PY
