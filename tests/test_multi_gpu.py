"""Real multi-GPU runs (one process per GPU, NVLink peers).  Skipped on a 1-GPU box."""
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(n: int, *args, timeout=600, script="mp_parity.py"):
    """torchrun on a free port; retried with a new port if the rendezvous lost a port race."""
    for _ in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(ROOT, "tests", script), *args]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
        if r.returncode == 0 or "EADDRINUSE" not in (r.stdout + r.stderr):
            return r
    return r


@pytest.mark.parametrize("G,config,extra", [
    (2, "tiny-skew", []), (2, "tiny", []), (4, "tiny-skew", []), (4, "tiny", ["--trace", "rotating-hot"]),
    (2, "gpt-small", ["--sampled", "--iters", "3"]), (8, "gpt-small", ["--sampled", "--iters", "3"]),
    (2, "medium", ["--dedup", "--iters", "4"]), (4, "medium", ["--dedup", "--iters", "4"]),
    (4, "tiny-skew", ["--dedup", "--trace", "rotating-hot"]),
    (4, "gpt-small", ["--dedup", "--sampled", "--iters", "3"]),
    (2, "tiny", ["--cf", "0.5"]), (4, "medium", ["--cf", "1.25", "--dedup", "--iters", "4"]),
    (4, "tiny-skew", ["--cf", "1.0", "--policy", "2"]),
    (4, "tiny-skew", ["--cf", "1.0", "--interval", "3", "--iters", "7", "--dedup"]),
    (2, "tiny", ["--tokens", "1"]), (4, "medium", ["--tokens", "0", "--cf", "1.25", "--iters", "3"]),
    (4, "tiny-skew", ["--tokens", "1", "--dedup", "--trace", "rotating-hot"]),
    (4, "medium", ["--host-state", "--dedup", "--iters", "4"]), (2, "medium", ["--host-state", "--iters", "3"]),
    (4, "medium", ["--dedup", "--lazy", "--iters", "4"]), (2, "tiny-skew", ["--dedup", "--lazy", "--tokens", "1"]),
    # ad-hoc random shapes (E, S per GPU, k, T, P, seed): ragged owner ranges, k = E, E = 1
    (2, "tiny", ["--adhoc", "7,5,3,602,528,11", "--dedup", "--lazy", "--cf", "0.8", "--tokens", "1"]),
    (4, "tiny", ["--adhoc", "13,4,2,1000,1344,12", "--dedup", "--tokens", "0"]),
    (4, "tiny", ["--adhoc", "3,3,3,404,96,13", "--policy", "1", "--interval", "2", "--iters", "5"]),
    (2, "tiny", ["--adhoc", "1,2,1,300,208,14", "--host-state"]),
    # update-stage edge values over NVLink: zero-token experts, +-0, denormals, overflow, NaN
    (2, "tiny-skew", ["--edge"]), (4, "medium", ["--edge", "--dedup", "--iters", "4"]),
    (4, "tiny-skew", ["--edge", "--host-state", "--dedup"]),
], ids=lambda x: "".join(a.lstrip("-") for a in x) if isinstance(x, list) else str(x))
def test_real_multi_gpu_parity(G, config, extra):
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    r = _torchrun(G, "--config", config, *extra)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


def test_missing_peer_times_out_instead_of_hanging():
    """Failure detection: a rank that skips an iteration -> MOE_ERR_TIMEOUT on its peer (~30 s)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    r = _torchrun(2, timeout=300, script="mp_failure.py")
    assert r.returncode == 0 and "mp_failure: OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("G,extra", [(2, ["--dedup", "--lazy", "--iters", "4"]), (4, ["--dedup", "--iters", "4", "--interval", "2"])])
def test_early_update_launch_real_mode(G, extra, monkeypatch):
    """The opt-in early update launch (MOE_EARLY_UPDATE=1) over NVLink: each rank's kernel
    acquires its own host's plan_{t+1} hand-off; bit-exact vs the oracle."""
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    monkeypatch.setenv("MOE_EARLY_UPDATE", "1")
    r = _torchrun(G, "--config", "medium", *extra)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.parametrize("G,extra", [(2, ["--dedup", "--lazy", "--iters", "4"]),
                                     (4, ["--dedup", "--iters", "4", "--cf", "1.25"])])
def test_fused_presum_real_mode(G, extra, monkeypatch):
    """The opt-in fused pre-sum (MOE_PRESUM_FUSED=1) over NVLink: partials released per GPU with
    system-scope flags, acquired by every owner before its first bulk pull; bit-exact."""
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    monkeypatch.setenv("MOE_PRESUM_FUSED", "1")
    r = _torchrun(G, "--config", "medium", *extra)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
