"""CPU-side checks of the C ABI: the library loads, exports every function include/dymoe.h
declares, validates arguments (naming the field) before touching the device, and its host-only
schedule helpers agree with the oracle.  No kernel is launched here."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import schedule as o_sched

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dymoe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(dymoe_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def d():
    from paper_2603_19172_b200 import build
    build.build()
    import paper_2603_19172_b200.dymoe as dm
    dm.lib()
    return dm


def test_exports_every_declared_symbol(d):
    names = declared_functions()
    assert len(names) >= 19
    raw = ctypes.CDLL(d.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), n
    assert set(names) == set(d.EXPORTED)


def test_version(d):
    assert b"sm_100a" in d.lib().dymoe_version()


def test_retention_and_tier_counts_match_oracle(d):
    for L in (1, 2, 3, 8, 32):
        for lam in np.linspace(0, 1, 11):
            for l in range(L):
                assert d.dymoe_retention_ratio(l, L, float(lam)) == pytest.approx(
                    o_sched.retention_ratio(l, L, float(lam)), abs=1e-15)
    for M in (1, 6, 8, 64, 256):
        for bits, lams in [((4, 2), (0.5,)), ((8, 4, 2), (0.25, 0.5)), ((4, 0), (0.0,)),
                           ((16, 8, 4, 2, 0), (0.0, 0.2, 0.2, 0.9))]:
            for clamp in (True, False):
                for l in range(32):
                    got = d.dymoe_tier_counts(l, 32, d.make_ladder(bits, lams, clamp_to_k=clamp), M, 2)
                    ref = o_sched.tier_counts(l, 32, o_sched.Ladder(bits, lams, clamp_to_k=clamp), M, 2)
                    assert got == ref


FAKE = ctypes.c_void_p(0x100000)   # never dereferenced: validation fails first


def _err(d, rc):
    return rc, d.lib().dymoe_last_error().decode()


def test_validation_messages_name_the_field(d):
    L = d.lib()
    rc, msg = _err(d, L.dymoe_route(FAKE, 4, 8, 9, FAKE, FAKE, None, None))
    assert rc == 1 and msg.startswith("k:")
    rc, msg = _err(d, L.dymoe_route(FAKE, 4, 300, 2, FAKE, FAKE, None, None))
    assert rc == 1 and msg.startswith("M:")
    rc, msg = _err(d, L.dymoe_quantize(FAKE, 4, 100, 4, 128, FAKE, FAKE, FAKE, None))
    assert rc == 1 and msg.startswith("K:")
    rc, msg = _err(d, L.dymoe_quantize(FAKE, 4, 128, 3, 128, FAKE, FAKE, FAKE, None))
    assert rc == 1 and msg.startswith("bits:")
    rc, msg = _err(d, L.dymoe_quantize(FAKE, 4, 128, 4, 64, FAKE, FAKE, FAKE, None))
    assert rc == 1 and msg.startswith("group:")
    lad = d.make_ladder((8, 4, 2), (0.6, 0.5))
    rc, msg = _err(d, L.dymoe_assign_bits(FAKE, 8, 0, 32, ctypes.byref(lad), 2, None, FAKE, None, None))
    assert rc == 1 and msg.startswith("ladder.lambdas")
    lad = d.make_ladder((4, 2), (0.5,))
    rc, msg = _err(d, L.dymoe_assign_bits(FAKE, 8, 32, 32, ctypes.byref(lad), 2, None, FAKE, None, None))
    assert rc == 1 and msg.startswith("layer:")
    lad = d.make_ladder((4, 2), (0.5,), m_active=True)
    rc, msg = _err(d, L.dymoe_assign_bits(FAKE, 8, 0, 32, ctypes.byref(lad), 2, None, FAKE, None, None))
    assert rc == 1 and msg.startswith("active_mask:")
    rc, msg = _err(d, L.dymoe_score(0, FAKE, 32, FAKE, None, 10, 8, 2, 11, FAKE, None, FAKE, None))
    assert rc == 1 and msg.startswith("k_tokens:")
    rc, msg = _err(d, L.dymoe_combine(FAKE, FAKE, FAKE, 3, 2, 6, 1, 7, FAKE, None))
    assert rc == 1 and (msg.startswith("Hd:") or msg.startswith("out_dtype:"))
    desc = d.LayerDesc(8, 2, 100, 256, None)
    h = ctypes.c_void_p()
    rc, msg = _err(d, L.dymoe_layer_create(ctypes.byref(desc), ctypes.byref(h)))
    assert rc == 1 and msg.startswith("desc.hidden:")


def test_no_cpu_fallback(d):
    import torch
    with pytest.raises(ValueError, match="CUDA"):
        d.dymoe_route(torch.zeros(2, 8), 2)


def test_ep_window_layout_and_validation(d):
    """Host-side parts of the peer-memory EP calls: the window size formula (flags, cnt[2][P][M],
    imp[2][P][M], red f32[2][64][Hd], recv_x bf16 and y_out f32 sections, each 256-byte aligned)
    and field-naming validation."""
    a = lambda v: (v + 255) // 256 * 256
    for P, M, Hd, cap in [(2, 8, 256, 64), (8, 64, 2048, 98304), (1, 1, 8, 0), (3, 7, 24, 5)]:
        want = (a(P * 4) + 2 * a(2 * P * M * 4) + a(2 * 64 * Hd * 4) + a(cap * Hd * 2)
                + a(cap * Hd * 4))
        assert d.dymoe_ep_window_bytes(P, M, Hd, cap) == want
    assert d.dymoe_ep_window_bytes(0, 8, 256, 4) == 0
    L = d.lib()
    w = d.EpWindow(4, 0, 2, 256, 16, 0, 0x100000)
    rc, msg = _err(d, L.dymoe_ep_publish_counts(ctypes.byref(w), FAKE, None))
    assert rc == 1 and msg.startswith("window.P:")
    w = d.EpWindow(2, 2, 8, 256, 16, 0, 0x100000)
    rc, msg = _err(d, L.dymoe_ep_barrier(ctypes.byref(w), 1, None, None))
    assert rc == 1 and msg.startswith("window.rank:")
    w = d.EpWindow(2, 0, 8, 100, 16, 0, 0x100000)
    rc, msg = _err(d, L.dymoe_ep_dispatch(ctypes.byref(w), FAKE, 4, FAKE, FAKE, FAKE, None, None))
    assert rc == 1 and msg.startswith("window.Hd:")
    w = d.EpWindow(2, 0, 8, 256, 16, 2, 0x100000)
    rc, msg = _err(d, L.dymoe_ep_combine(ctypes.byref(w), FAKE, FAKE, 4, 2, FAKE, 1, 0, FAKE, None, None))
    assert rc == 1 and msg.startswith("window.parity:")
    w = d.EpWindow(2, 0, 8, 256, 16, 0, None)
    rc, msg = _err(d, L.dymoe_ep_combine(ctypes.byref(w), FAKE, FAKE, 4, 2, FAKE, 1, 0, FAKE, None, None))
    assert rc == 1 and msg.startswith("window.peers:")


def test_ep_handle_validation(d):
    """dymoe_ep_create validates its configuration without touching the device (field named)."""
    L = d.lib()
    h = ctypes.c_void_p()
    cfg = d.EpConfig(8, 2, 256, 512, 16, d.DYMOE_EP_PEER)
    rc, msg = _err(d, L.dymoe_ep_create(0, 9, None, ctypes.byref(cfg), ctypes.byref(h)))
    assert rc == 1 and msg.startswith("world:")
    rc, msg = _err(d, L.dymoe_ep_create(2, 2, None, ctypes.byref(cfg), ctypes.byref(h)))
    assert rc == 1 and msg.startswith("rank:")
    bad = d.EpConfig(8, 2, 200, 512, 16, d.DYMOE_EP_PEER)
    rc, msg = _err(d, L.dymoe_ep_create(0, 2, None, ctypes.byref(bad), ctypes.byref(h)))
    assert rc == 1 and msg.startswith("cfg.hidden:")
    bad = d.EpConfig(8, 2, 256, 512, 16, 0)
    rc, msg = _err(d, L.dymoe_ep_create(0, 2, None, ctypes.byref(bad), ctypes.byref(h)))
    assert rc == 1 and msg.startswith("cfg.transports:")
    nccl = d.EpConfig(8, 2, 256, 512, 16, d.DYMOE_EP_NCCL)
    rc, msg = _err(d, L.dymoe_ep_create(0, 2, None, ctypes.byref(nccl), ctypes.byref(h)))
    assert rc == 1 and msg.startswith("nccl_uid:")
    rc, msg = _err(d, L.dymoe_moe_forward_ep(None, None, 1, 0, None, None, 0, 0, None, None, None, 0, None))
    assert rc == 1 and msg.startswith("ep:")
    assert L.dymoe_ep_workspace_size(None, 4, 0, 0) == 0


def test_ep_unique_id_is_ncclish(d):
    """The NCCL unique id comes from the NCCL library the process loads (no device needed)."""
    import paper_2603_19172_b200.ep as ep
    a, b = ep.unique_id(), ep.unique_id()
    assert len(a) == d.EP_UID_BYTES and a != b
