"""Memory and race checks without compute-sanitizer (closed on this GPU pool: runs under it left
GPUs needing a reset).  Three substitutes, over small cases of every kernel family:

* FMM_GUARD=1: every device buffer a context allocates carries a 4 KiB guard zone after its usable
  bytes; fmm_debug_check verifies every zone after the run (an out-of-bounds write past any
  buffer's end is caught);
* FMM_POISON=1: fresh allocations are filled with 0xFF bytes (NaN floats, huge indices), and the
  results must still match the oracle bit for bit (structure) and to tolerance (fields): a kernel
  that reads memory no kernel wrote would carry the poison into them;
* repeated solves on one context must be bitwise identical (a shared-memory or look-back race in the
  sort, the traversal, the TMA/mbarrier P2P pipeline or the M2L would show up as run-to-run
  differences).
"""
import numpy as np
import pytest

import oracle
import synth
from fieldcheck import assert_fields

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1405_7487_b200 import build
    build.build()
    return torch


CASES = [("cube", 1 << 15, 10, 0.4, 64, "f32"),      # c2-shaped: mid leaves (TMA P2P), mirror M2L
         ("plummer", 20000, 10, 0.4, 64, "f32"),     # adaptive: every P2P leaf class, deep lists
         ("sphere", 20000, 10, 0.4, 512, "f32"),     # big leaves
         ("plummer", 6000, 6, 0.4, 16, "f64")]       # fp64 kernels


@pytest.mark.parametrize("kind,n,P,theta,ncrit,prec", CASES)
def test_guard_and_poison(torch_cuda, monkeypatch, kind, n, P, theta, ncrit, prec):
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    monkeypatch.setenv("FMM_GUARD", "1")
    monkeypatch.setenv("FMM_POISON", "1")
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate(kind, n, 900 + n, dt)
    f = FMM(n, P, theta, ncrit, prec)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    outs = []
    for _ in range(4):     # first build, the size-learning rebuilds
        phi, grad = f.solve(tp, tq)
        outs.append((phi.cpu().numpy(), grad.cpu().numpy()))
    f.build(tp)
    outs.append(tuple(x.cpu().numpy() for x in f.evaluate(tp, tq)))
    assert f.debug_check() == 0
    for a, b in outs[1:]:
        np.testing.assert_array_equal(a, outs[0][0])
        np.testing.assert_array_equal(b, outs[0][1])
    o = oracle.FMM(pos.astype(np.float64), q.astype(np.float64), P, theta, ncrit).traverse()
    gm, gp = f.lists()
    om, op = o.lists()
    np.testing.assert_array_equal(gm, om)
    np.testing.assert_array_equal(gp, op)
    ophi, ograd = o.evaluate()
    assert_fields(outs[0][0], ophi, outs[0][1], ograd, TOL[prec], kind)


def test_guard_dist_and_debug_stages(torch_cuda, monkeypatch):
    """The distributed driver (in-process group, 3 ranks, both partitioners; the ORB run with the
    split interactions of FMM_DIST_SPLIT=1) and the debug stage entries under guard zones and
    poisoned allocations."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    from paper_1405_7487_b200.dist import DistFMM, LocalGroup, run_ranks
    monkeypatch.setenv("FMM_GUARD", "1")
    monkeypatch.setenv("FMM_POISON", "1")
    n, K = 15000, 3
    pos, q = synth.generate("plummer", n, 31, np.float32)
    cuts = np.linspace(0, n, K + 1).astype(int)
    P_in = [torch.from_numpy(pos[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    Q_in = [torch.from_numpy(q[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    for part in ("morton", "orb"):
        monkeypatch.setenv("FMM_DIST_SPLIT", "1" if part == "orb" else "0")
        G = LocalGroup(K)
        Ds = [DistFMM(n, 10, 0.4, 64, "f32", 0, K, r, group=G, partitioner=part) for r in range(K)]
        streams = [torch.cuda.Stream() for _ in range(K)]
        res = []
        for _ in range(2):
            out = run_ranks(lambda r: Ds[r].solve(P_in[r], Q_in[r], int(cuts[r]), reuse_weights=True,
                                                  stream=streams[r]), K)
            torch.cuda.synchronize()
            res.append(np.concatenate([o[0].cpu().numpy() for o in out]))
        for D in Ds:
            assert D.debug_check() == 0
        t = synth.sample_targets(n, 300, 31)
        dp, _ = oracle.direct(pos.astype(np.float64), q.astype(np.float64), t)
        assert oracle.rel_l2(res[1][t], dp) < 1e-3
        for D in Ds:
            D.close()
        G.close()
    f = FMM(n, 6, 0.5, 16, "f64")
    p64, q64 = pos.astype(np.float64), q.astype(np.float64)
    o = oracle.FMM(p64, q64, 6, 0.5, 16).traverse()
    o.evaluate()
    _, perm = o.sorted()
    cells = o.cells()
    m2l, p2p = o.lists()
    M, _ = o.expansions()
    cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    i32 = lambda x: cu(x.astype(np.int32))  # noqa: E731
    f.debug_p2p(cu(p64[perm]), cu(q64[perm]), i32(cells["body_begin"]), i32(cells["body_count"]),
                i32(cells["child_count"]), i32(p2p))
    f.debug_m2l(cu(cells["center"]), cu(cells["level"]), cu(M), 50.0, i32(m2l))
    assert f.debug_check() == 0
