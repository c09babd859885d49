"""bench.py's N > 1 code path (row slabs, halo lists over torch.distributed,
the library's NCCL halo exchange and reductions, max-over-ranks timing, the
JSON line) launched exactly as the driver launches it -- torchrun, one process
per rank -- but with every rank on GPU 0 and the library linked against the
test stand-in for NCCL (bench.py --test-fake-nccl, tests/native/fake_nccl.cpp).
The sharded run must take the same number of iterations and mat-vecs as the
single-process run of the same workload."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(n, extra):
    args = ["bench.py", "--gpus", str(n), "--steps", "2", "--warmup", "3", "--no-profile",
            "--no-cpu-baseline", *extra]
    if n > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
               str(_free_port()), *args, "--test-fake-nccl"]
    else:
        cmd = [sys.executable, *args]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]       # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("extra", [
    # NCCL code path (the test stand-in for NCCL)
    ["--config", "C3s", "--deg", "10", "--comm", "nccl"],             # real, Chebyshev, Lanczos
    ["--config", "C5s", "--deg", "16", "--comm", "nccl"],             # complex, sharded Ritz setup, CGS2
    ["--config", "C7s", "--deg", "7", "--check-every", "4", "--comm", "nccl"],  # power-law graph slabs
    # peer memory (the default: CUDA IPC windows between the rank processes)
    ["--config", "C4s", "--deg", "20"],
    ["--config", "C5s", "--deg", "16"],
], ids=["c3s_nccl", "c5s_nccl", "c7s_nccl", "c4s_peer", "c5s_peer"])
def test_bench_two_ranks_matches_one(extra):
    one = _bench(1, extra)
    two = _bench(2, extra)
    assert two["n_gpus"] == 2 and "test_mode" in two
    assert two["layout"]["ranks_joined"] == 2
    assert two["config"]["parallelism"].startswith("row slabs x2")
    assert ("NCCL" if "nccl" in extra else "peer-memory") in two["config"]["parallelism"]
    assert two["config"]["m"] == one["config"]["m"]
    assert two["config"]["mvms"] == one["config"]["mvms"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0 and two["gpu_launches"] > 0
