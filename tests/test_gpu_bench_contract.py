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


def test_ep_two_ranks_line_with_p2p():
    """N = 2 bench path (two processes time-sharing the one GPU over gloo -- a test hook, never a
    reported number): the EP line, the replicated-decode and the peer-memory variants."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29641", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--copies", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["scaling"] == "weak"
    assert j["ep_replicated_decode"]["value"] > 0
    p = j["ep_p2p"]
    assert "error" not in p, p
    assert p["value"] > 0 and p["status"] == 0 and p["barrier"] == "host"


def test_ep_two_ranks_p2p_main_line():
    """The N = 2 main line on the peer-memory path (forced under the gloo test hook), e2e included."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29643", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--copies", "1",
           "--ep-main", "p2p", "--workload", "finegrained", "--tokens", "256"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["ep_path"] == "p2p" and j["value"] == j["ep_p2p"]["value"] and j["e2e"]["value"] > 0
    assert j["ep_nccl_all_to_all"]["value"] > 0 and "peer-memory" in j["config"]["parallelism"]
