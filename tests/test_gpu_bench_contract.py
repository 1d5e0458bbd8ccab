"""The bench.py JSON-line contract (driver-facing), on a short run: every required key, sane
values, the roofline / e2e / clocks / cpu_baseline objects, and the stack workload line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def _common(j):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "clocks", "e2e", "gpu_launches"):
        assert k in j, k
    assert j["value"] > 0 and j["ms_per_step"] > 0 and j["n_gpus"] == 1 and j["warmup"] >= 3
    assert j["higher_is_better"] is True and j["vs_baseline"] is None
    r = j["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] < 1.2 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] > 0 and "sm_mhz" in j["clocks"] and "reasons" in j["clocks"]
    assert "workload" in j["config"]


def test_decode_line_with_cpu_baseline():
    j = _run("--steps", "8", "--warmup", "3", "--copies", "1")
    _common(j)
    assert j["config"]["workload"] == "mixtral_decode" and j["roofline"]["bound"] == "hbm"
    assert j["roofline"]["traffic"] is None or j["roofline"]["traffic"] > 0
    cb = j["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    assert set(j["quantize"]) >= {"int8", "int4", "int2"}


def test_stack_line():
    j = _run("--workload", "stack", "--steps", "2", "--warmup", "3")
    _common(j)
    assert j["config"]["workload"] == "mixtral_stack32_decode" and j["config"]["layers"] == 32


def test_decode_line_sub_lines():
    """The default line carries the rest of the metric: prefill with its own e2e
    and tensor roofline, decode B = 1, the paper's 4/2 and 4/0 ladders, the per-width sweep."""
    j = _run("--steps", "6", "--warmup", "3", "--copies", "1", "--no-cpu-baseline")
    subs = j["sub_lines"]
    p = subs["prefill"]
    assert p["tokens_per_step"] == 2048 and p["roofline"]["bound"] == "tensor" and p["e2e"]["value"] > 0
    assert subs["decode_b1"]["tokens_per_step"] == 1 and subs["decode_b1"]["roofline"]["bound"] == "hbm"
    for k in ("decode_b1_ladder_4_2", "decode_b8_ladder_4_2", "decode_b1_ladder_4_0", "decode_b8_ladder_4_0"):
        assert subs[k]["value"] > 0, k
    assert set(subs["decode_b8_ladder_4_2"]["widths_active"]) <= {"4", "2"}
    sw = subs["decode_width_sweep"]
    for w in ("bf16", "int8", "int4", "int2"):
        assert 0 < sw[w]["w13_frac"] < 1.2 and 0 < sw[w]["w2_frac"] < 1.2


def _ep_line(*extra, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--copies", "1",
           *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_ep_two_ranks_line():
    """N = 2 bench path (two processes time-sharing the one GPU, gloo for the plumbing -- a test
    hook, never a reported number): the C-ABI EP layer over peer windows (CUDA IPC), e2e and the
    replicated-decode placement."""
    j = _ep_line(port=29641)
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["scaling"] == "weak"
    assert j["ep_path"] == "peer" and j["ep_transports"]["peer"]["status"] == 0
    assert j["e2e"]["value"] > 0 and j["gpu_launches"] > 0
    assert j["ep_replicated_decode"]["peer"]["value"] > 0


def test_ep_two_ranks_finegrained_prefill():
    j = _ep_line("--workload", "finegrained", "--tokens", "256", port=29643)
    assert j["config"]["workload"] == "finegrained_prefill" and j["roofline"]["bound"] == "tensor"
    assert j["value"] > 0 and j["ep_transports"]["peer"]["status"] == 0


def test_gpus_flag_self_launches():
    """`python bench.py --gpus 2` without torchrun launches the two ranks itself (n_gpus == 2)."""
    j = _run("--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--copies", "1")
    assert j["n_gpus"] == 2 and j["value"] > 0
