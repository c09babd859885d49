"""Peer-memory communication (ppf_mat_peer_window / ppf_mat_peer_connect,
csrc/peer.cu; SURVEY §8(e) "direct peer loads/stores over NVLink"): every
halo exchange is a push kernel storing boundary entries straight into the
neighbour's receive slot + a system-scope arrival counter, every reduction a
store of the partials into every rank's window + a rank-order sum.

With one GPU the ranks are emulated as R contexts of ONE (child) process, each
on its own CUDA stream and host thread, their windows plain device pointers of the
same process (ppf_mat_peer_connect maps a same-process descriptor by pointer,
another process's by CUDA IPC).  No kernel waits on another: the waits are
stream front-end waits (cuStreamWaitValue32) on the rank's own counters, so
the ranks never compete for SMs while waiting (B200_PROFILING.md: with fewer
GPUs than ranks, no spinning kernels).  The gathered slabs must match the
single-process oracle like the NCCL / host-transport runs of
test_gpu_multirank.py, and the peer reductions are bit-identical on all ranks
(rank-order sums), which the identical iteration counts and H check."""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

from inputs import configs
from tests.test_gpu_multirank import CASES, WORLD, X_TOL, _slab_bounds, oracle_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


CHILD_ENV = {
    # every emulated rank's streams on a hardware queue of its own: a stream
    # parked in a peer wait must not hold up, behind it in a shared queue, the
    # stream whose push releases it (CUDA maps streams onto this many queues)
    "CUDA_DEVICE_MAX_CONNECTIONS": "32",
}


def _raw_stream():
    """A fresh non-blocking stream (not from torch's pre-created pool)."""
    import ctypes as C
    cudart = C.CDLL("libcudart.so.12")
    h = C.c_void_p()
    assert cudart.cudaStreamCreateWithFlags(C.byref(h), 1) == 0
    return torch.cuda.ExternalStream(h.value)


def _make_ranks(A, b, cfg, world):
    import paper_2401_06684_b200 as pp
    bounds = _slab_bounds(cfg, A.n, world)
    plans = []
    for r in range(world):
        lo, hi = bounds[r], bounds[r + 1]
        rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
        sl = slice(int(A.row_ptr[lo]), int(A.row_ptr[hi]))
        plans.append(pp.Plan(rp, A.col[sl], A.val[sl], row_bounds=bounds, rank=r))
    needs = [{p: plans[r].halo_recv(p) for p in range(world)} for r in range(world)]
    for r in range(world):
        for p in range(world):
            plans[r].set_halo_send(p, needs[p][r] - bounds[r])
    ranks = []
    for r in range(world):
        st = _raw_stream()
        ctx = pp.Context(0, rank=r, nranks=world, stream=st)
        M = pp.Matrix(ctx, plans[r])
        bd = torch.from_numpy(np.ascontiguousarray(b[bounds[r]:bounds[r + 1]])).cuda()
        ranks.append(dict(ctx=ctx, M=M, bd=bd, st=st))
    descs = [R["M"].peer_window() for R in ranks]
    for R in ranks:
        R["M"].peer_connect(descs)
    return bounds, ranks


def _run_threads(fn, ranks, timeout=240):
    """One host thread per rank.  Inside `fn` only library calls on memory
    allocated beforehand: no torch kernels (a first launch loads its module)
    and no allocations (device / pinned allocation synchronises the device),
    either of which would wait for a stream parked in a peer wait."""
    errs = [None] * len(ranks)

    def body(r):
        try:
            fn(r, ranks[r])
            ranks[r]["st"].synchronize()
        except BaseException as e:  # noqa: BLE001 -- re-raised in the main thread
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(ranks))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
        if t.is_alive():
            print("a rank did not finish (peer exchange stalled)", flush=True)
            for r, e in enumerate(errs):   # a rank that failed leaves the others waiting
                if e is not None:
                    print(f"rank {r} failed: {e!r}", flush=True)
            os._exit(3)   # tear the context down instead of hanging
    for e in errs:
        if e is not None:
            raise e


def child_run(case, q_path, out_path, world=None, graphs=False):
    """Child process: the case on `world` emulated ranks with peer memory,
    launched directly (graphs=False): ranks emulated as threads of one process
    cannot replay captured graphs whose stream waits depend on each other --
    the graphs' internal streams share hardware queues, so one rank's wait node
    can block another rank's push (measured: a stall).  The graph path is
    tested between processes (test_gpu_multirank.py::test_peer_ipc_graph_replay_bitwise)."""
    import paper_2401_06684_b200 as pp
    name, deg, kw = CASES[case]
    cfg = configs.CONFIGS[name]
    world = world or WORLD.get(case, 2)
    A, b, iv = configs.build(name)
    _, ranks = _make_ranks(A, b, cfg, world)
    for R in ranks:
        R["ctx"].set_graphs(graphs)
    power = 2 if cfg.func == "sign" else 1
    for R in ranks:
        if cfg.poly == "ritz":
            qd = np.load(q_path)
            R["q"] = pp.Poly.newton(qd[0], qd[1])
            if cfg.params.get("ritz_start") == "Ab":
                R["q"].set_newton_eval("basis")
            R["start"] = torch.empty_like(R["bd"])
            R["rwork"] = pp.Poly.ritz_workspace(R["ctx"], R["M"], deg)
        else:
            R["q"] = pp.Poly.chebyshev(*iv, deg)
        opts = pp.api.make_opts(func=cfg.func, m_max=cfg.m_max, tol=cfg.tol, **kw)
        R["work"] = pp.api.Workspace(R["ctx"], R["M"], R["q"], opts)
        R["x"] = torch.empty_like(R["bd"])
    torch.cuda.synchronize()

    def body(r, R):
        if cfg.poly == "ritz":   # the sharded Ritz setup, through peer memory too
            start = R["bd"]
            if cfg.params.get("ritz_start") == "Ab":
                R["M"].spmv(R["bd"], R["start"])
                start = R["start"]
            R["nodes"] = pp.Poly.ritz_newton(R["ctx"], R["M"], start, deg, power=power,
                                             work=R["rwork"]).export()["nodes"]
        R["x"], R["rep"] = pp.run(R["ctx"], R["M"], R["q"], R["bd"], x=R["x"], work=R["work"],
                                  func=cfg.func, m_max=cfg.m_max, tol=cfg.tol, **kw)
        R["H"] = pp.api.hessenberg(R["ctx"], cfg.complex_)[0]

    _run_threads(body, ranks)
    out = dict(x=np.concatenate([R["x"].cpu().numpy() for R in ranks]),
               m=np.array([R["rep"].iterations for R in ranks]),
               H=np.stack([R["H"] for R in ranks]))
    if cfg.poly == "ritz":
        out["nodes"] = np.stack([R["nodes"] for R in ranks])
    np.savez(out_path, **out)


def child_spmv(out_path, steps=100):
    """Child process: `steps` back-to-back sharded SpMVs y_{k+1} = A y_k on 3
    emulated ranks (each receive slot reused steps/2 times)."""
    import paper_2401_06684_b200 as pp
    name = "C3s"
    cfg = configs.CONFIGS[name]
    A, b, _ = configs.build(name)
    bounds, ranks = _make_ranks(A, b, cfg, 3)
    for R in ranks:
        R["y"] = [R["bd"]] + [torch.empty_like(R["bd"]) for _ in range(steps)]
    torch.cuda.synchronize()

    def body(r, R):
        for k in range(steps):
            R["M"].spmv(R["y"][k], R["y"][k + 1])

    _run_threads(body, ranks)
    ys = np.stack([np.concatenate([R["y"][k].cpu().numpy() for R in ranks])
                   for k in range(steps + 1)])
    np.save(out_path, ys)


def _child(call):
    env = dict(os.environ, **CHILD_ENV)
    r = subprocess.run([sys.executable, "-c", "import tests.test_gpu_peer as t; t." + call],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


# (case, ranks): every sharded case at its usual rank count, plus the 8-rank
# layout of an 8-GPU node (C3s: 30 planes -> slabs of 3-4 planes; C5s: a ring of
# 4 time slices -> 4 ranks, each with two neighbours)
PEER_RUNS = [(c, WORLD.get(c, 2)) for c in CASES] + [("c3s_lanczos", 8), ("c4s_cgs2_sqrt", 8),
                                                      ("c5s_ritz", 4)]


@pytest.mark.parametrize("case,world", PEER_RUNS)
def test_peer_ranks_match_oracle(case, world, tmp_path):
    assert torch.cuda.is_available(), "GPU tests need a B200"
    cfg, A, b, iv, qo, res = oracle_case(case)
    q_path, out = str(tmp_path / "q.npy"), str(tmp_path / "out.npz")
    if cfg.poly == "ritz":
        np.save(q_path, np.stack([qo.nodes, qo.dd]))
    _child(f"child_run({case!r}, {q_path!r}, {out!r}, {world})")
    o = np.load(out)
    assert all(int(m) == res.m for m in o["m"])               # every rank, the oracle's m
    assert all(np.array_equal(H, o["H"][0]) for H in o["H"])  # rank-order sums: identical H
    if cfg.poly == "ritz":
        for nodes in o["nodes"]:
            assert np.abs(np.sort_complex(nodes) - np.sort_complex(qo.nodes)).max() < 1e-8
    err = np.linalg.norm(o["x"] - res.x) / np.linalg.norm(res.x)
    if err > X_TOL:   # which slabs are off (diagnostic)
        name = CASES[case][0]
        bounds = _slab_bounds(configs.CONFIGS[name], len(res.x), world)
        per = [float(np.linalg.norm((o["x"] - res.x)[lo:hi]) / np.linalg.norm(res.x[lo:hi]))
               for lo, hi in zip(bounds[:-1], bounds[1:])]
        pytest.fail(f"x rel. error {err:.3g}; per slab {per}")


def test_peer_spmv_many_epochs(tmp_path):
    """Back-to-back sharded SpMVs (the receive slots reused many times, ranks
    free to drift apart by one slot) equal the unsharded products up to the
    order in which the halo block is added (diagonal block first)."""
    from oracle.spmv import Operator
    out = str(tmp_path / "y.npy")
    _child(f"child_spmv({out!r})")
    ys = np.load(out)
    A, b, _ = configs.build("C3s")
    op = Operator(A.to_scipy())
    y = b.copy()
    for k in range(1, ys.shape[0]):
        y = op.matvec(y)
        assert np.linalg.norm(ys[k] - y) <= 1e-13 * k * np.linalg.norm(y), k


def test_peer_window_errors():
    """ppf_mat_peer_window / _connect argument checking (include/ppf.h): a
    single-rank matrix has no window; descriptors must come in rank order with
    matching halo counts; connect needs a window and happens once; a matrix
    disconnected again has no transport left (ppf_run: PPF_ESTATE)."""
    import paper_2401_06684_b200 as pp
    from paper_2401_06684_b200._lib import PPFError
    name = "C3s"
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    ctx1 = pp.Context(0)
    M1 = pp.Matrix(ctx1, pp.Plan.from_csr(A))
    with pytest.raises(PPFError, match="EINVAL"):
        M1.peer_window()
    bounds, ranks = _make_ranks(A, b, cfg, 2)           # connected, same process
    d0, d1 = ranks[0]["M"].peer_window(), ranks[1]["M"].peer_window()   # fresh windows
    with pytest.raises(PPFError, match="EINVAL"):
        ranks[0]["M"].peer_connect([d1, d0])               # not in rank order
    with pytest.raises(PPFError, match="EINVAL"):
        ranks[0]["M"].peer_connect([d0, d0])               # rank 1's slot holds rank 0's descriptor
    ranks[0]["M"].peer_connect([d0, d1])
    with pytest.raises(PPFError, match="EINVAL"):
        ranks[0]["M"].peer_connect([d0, d1])               # already connected
    ranks[0]["M"].peer_connect(None)                       # back to no transport
    q = pp.Poly.chebyshev(*iv, 4)
    with pytest.raises(PPFError, match="ESTATE"):
        pp.run(ranks[0]["ctx"], ranks[0]["M"], q, ranks[0]["bd"], func=cfg.func, m_max=5,
               stop="fixed")
