python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import synthetic, bench
import paper_2603_19172_b200.dymoe as d
d.lib()
dev = torch.device('cuda')
cfg = synthetic.CONFIGS['mixtral_prefill']
layers = bench.build_layer_copies(d, cfg, 2, dev)
lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
x, lg, a = synthetic.layer_inputs(cfg, 5, dev)
for b in (16, 8, 4, 2):
    forced = torch.full((8,), b, dtype=torch.uint8, device=dev)
    ws = [L.workspace(cfg.T, dev) for L, _ in layers]
    for i in range(3): layers[i % 2][0].forward(x, lg, lad, 0, 32, phase=d.DYMOE_PREFILL, attn_mass=a, forced_bits=forced, ws=ws[i % 2])
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(8)]
    for r in evs:
        for e in r: e.record()
    for i in range(8):
        layers[i % 2][0].forward(x, lg, lad, 0, 32, phase=d.DYMOE_PREFILL, attn_mass=a, forced_bits=forced, ws=ws[i % 2], prof_events=evs[i])
    torch.cuda.synchronize()
    off = layers[0][0].views(cfg.T, ws[0])['expert_off'].cpu()
    n = int(off[-1])
    fl = 6.0 * cfg.hidden * cfg.ffn * n
    t13 = sum(e[0].elapsed_time(e[1]) for e in evs) / 8 / 1e3
    t2 = sum(e[1].elapsed_time(e[2]) for e in evs) / 8 / 1e3
    print('bits', b, 'W13 %.0f TF/s  W2 %.0f TF/s  rows %d' % (fl * 2 / 3 / t13 / 1e12, fl / 3 / t2 / 1e12, n), flush=True)
PY
python tools/profile_step.py --workload prefill --layer 20 --input 4 --warmup 1 > gpurun_out/r01_step_prefill.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefill_gemm -s 2 -c 2 -o gpurun_out/r01_prefill_full -f python tools/profile_step.py --workload prefill --layer 20 --input 4 --warmup 1 > gpurun_out/ncu_pf.log 2>&1
tail -1 gpurun_out/ncu_pf.log
