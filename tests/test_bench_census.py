"""bench.py's algorithmic work per step (the roofline numerators, DESIGN.md §7 / SURVEY §8d) against
the formulas written out by hand for small cases."""
import numpy as np

import bench
import synthetic


def test_bytes_per_weight():
    assert bench.bytes_per_weight(16) == 2.0
    for b in (8, 4, 2):
        assert bench.bytes_per_weight(b) == b / 8 + 5 / 128     # codes + fp32 scale + u8 zero per 128


def test_algorithmic_bytes_hand_case():
    cfg = synthetic.MoEConfig("c", M=4, k=2, hidden=256, ffn=512, T=3)
    bits = np.array([8, 0, 2, 16], np.uint8)
    off = np.array([0, 2, 3, 3, 6])            # rows per expert 2, 1 (skipped), 0, 3
    b13, b2 = bench.algorithmic_bytes(cfg, bits, off)
    Hd, F = 256, 512
    w8, w16 = 1 + 5 / 128, 2.0
    e13 = (2 * F * Hd * w8 + 2 * Hd * 2 + 2 * F * 2) + (2 * F * Hd * w16 + 3 * Hd * 2 + 3 * F * 2)
    e2 = (Hd * F * w8 + 2 * F * 2 + 2 * Hd * 4) + (Hd * F * w16 + 3 * F * 2 + 3 * Hd * 4)
    assert b13 == e13 and b2 == e2


def test_algorithmic_flops_counts_executed_pairs_only():
    cfg = synthetic.MoEConfig("c", M=4, k=2, hidden=256, ffn=512, T=3)
    bits = np.array([8, 0, 2, 16], np.uint8)
    off = np.array([0, 2, 3, 3, 6])
    assert bench.algorithmic_flops(cfg, off, bits) == 6.0 * 256 * 512 * (2 + 0 + 0 + 3)


def test_workload_configs_match_baseline_configs():
    """bench.py workloads -> BASELINE.json configs: [1] Mixtral decode (B tokens), [2] Mixtral
    prefill 2048, [3]'s fine-grained layer (64 experts, top-6, hidden 2048, ffn 1408)."""
    import argparse
    for w, (M, k, Hd, F, T, dec, name) in {
            "decode": (8, 2, 4096, 14336, 8, True, "mixtral_decode"),
            "prefill": (8, 2, 4096, 14336, 2048, False, "mixtral_prefill"),
            "finegrained": (64, 6, 2048, 1408, 2048, False, "finegrained_prefill"),
            "finegrained_decode": (64, 6, 2048, 1408, 8, True, "finegrained_decode")}.items():
        cfg, is_dec, wname = bench.workload_cfg(argparse.Namespace(workload=w, batch=8, tokens=2048))
        assert (cfg.M, cfg.k, cfg.hidden, cfg.ffn, cfg.T, is_dec, wname) == (M, k, Hd, F, T, dec, name)
