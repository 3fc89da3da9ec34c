"""GPU (libfmm, sm_100a) versus the CPU oracle, through the C-ABI.

Bar (north_star): keys, permutation, cells, fp64 geometry and the canonical
M2L/P2P lists bit-exact; phi and grad relative L2 <= 1e-12 in fp64, <= 1e-5 in fp32.
"""
import numpy as np
import pytest

import oracle
import synth
from fieldcheck import assert_field, assert_fields

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


def run_gpu(torch, pos, q, P, theta, ncrit, prec):
    from paper_1405_7487_b200 import FMM
    f = FMM(max(len(pos), 1), P, theta, ncrit, prec)
    dt = torch.float32 if prec == "f32" else torch.float64
    tp = torch.from_numpy(np.ascontiguousarray(pos)).to(dt).cuda()
    tq = torch.from_numpy(np.ascontiguousarray(q)).to(dt).cuda()
    phi, grad = f.solve(tp, tq)
    torch.cuda.synchronize()
    return f, phi.cpu().numpy().astype(np.float64), grad.cpu().numpy().astype(np.float64)


def check_structure(f, o):
    assert f.counts()["ncell"] == o.counts()["ncell"]
    gk, gp = f.sorted()
    ok, op = o.sorted()
    np.testing.assert_array_equal(gk, ok)
    np.testing.assert_array_equal(gp, op)
    gc, oc = f.cells(), o.cells()
    for k in oc:
        np.testing.assert_array_equal(gc[k], oc[k], err_msg=k)
    gm, gpl = f.lists()
    om, opl = o.lists()
    np.testing.assert_array_equal(gm, om)
    np.testing.assert_array_equal(gpl, opl)
    gcnt, ocnt = f.counts(), o.counts()
    for k in ("nleaf", "depth", "n_m2l", "n_p2p", "p2p_interactions"):
        assert gcnt[k] == ocnt[k], k


CASES = [
    # kind, n, P, theta, ncrit, prec
    ("cube", 4096, 4, 0.5, 32, "f64"),       # BASELINE configs[0]
    ("cube", 4133, 4, 0.5, 32, "f32"),       # ragged tail over several sort tiles
    ("plummer", 3000, 6, 0.4, 16, "f64"),
    ("plummer", 5000, 10, 0.4, 64, "f32"),
    ("sphere", 2000, 5, 0.6, 8, "f64"),
    ("cube", 1000, 1, 0.3, 8, "f64"),        # P = 1: monopole only, no far gradient
    ("cube", 1000, 2, 0.7, 1, "f64"),        # ncrit = 1
    ("cube", 700, 16, 0.5, 32, "f64"),       # maximum P
    ("plummer", 3000, 12, 0.5, 32, "f32"),   # fp32 register M2L past P = 10 (configs[4] P sweep)
    ("cube", 2500, 16, 0.5, 32, "f32"),
    ("plummer", 64, 3, 0.5, 64, "f32"),      # single leaf = direct sum
    ("cube", 7, 4, 0.5, 2, "f64"),
    ("sphere", 30000, 10, 0.4, 512, "f32"),  # Table I case 2 parameters (ncrit 512 leaves)
]


@pytest.mark.parametrize("kind,n,P,theta,ncrit,prec", CASES)
def test_parity_small(torch_cuda, kind, n, P, theta, ncrit, prec):
    pos, q = synth.generate(kind, n, 100 + n, np.float32 if prec == "f32" else np.float64)
    f, phi, grad = run_gpu(torch_cuda, pos, q, P, theta, ncrit, prec)
    o = oracle.FMM(pos.astype(np.float64), q.astype(np.float64), P, theta, ncrit).traverse()
    check_structure(f, o)
    ophi, ograd = o.evaluate()
    assert_fields(phi, ophi, grad, ograd, TOL[prec], f"{kind} n={n} P={P}")
    if prec == "f64":
        gM, gL = f.expansions()
        oM, oL = o.expansions()
        assert np.abs(gM - oM).max() <= 1e-12 * max(np.abs(oM).max(), 1e-300)
        assert np.abs(gL - oL).max() <= 1e-11 * max(np.abs(oL).max(), 1e-300)


@pytest.mark.parametrize("prec,P", [("f64", 2), ("f32", 4)])
def test_long_list_segments(torch_cuda, prec, P):
    # tiny theta and ncrit on a Plummer cloud: M2L segments of ~8.8k sources and a P2P segment
    # of ~23.7k source leaves exercise the big-segment sort path (> 4096 per target)
    pos, q = synth.generate("plummer", 30000, 7, np.float32 if prec == "f32" else np.float64)
    f, phi, grad = run_gpu(torch_cuda, pos, q, P, 0.2, 2, prec)
    o = oracle.FMM(pos.astype(np.float64), q.astype(np.float64), P, 0.2, 2).traverse()
    check_structure(f, o)
    m, p2 = o.lists()
    assert np.bincount(m[:, 0]).max() > 4096 and np.bincount(p2[:, 0]).max() > 4096
    t = synth.sample_targets(30000, 300, 7)
    ophi, ograd = o.evaluate(t)
    assert_fields(phi[t], ophi, grad[t], ograd, TOL[prec])


@pytest.mark.parametrize("prec,P", [("f64", 4), ("f32", 10)])
def test_duplicates_and_coincident(torch_cuda, prec, P):
    """Coincident points: a single-child chain to level 21, so M2L pairs span > 14 levels -- in
    fp32 the 2^(level gap) operand scale of the register kernels would leave the fp32 exponent
    range, and m2l_pass routes such trees to the fp64 kernel."""
    pos, q = synth.generate("cube", 300, 5)
    pos = np.vstack([pos, pos[:50], np.full((40, 3), 0.125)])
    q = np.concatenate([q, q[:50], np.linspace(-1, 1, 40)])
    if prec == "f32":
        pos = pos.astype(np.float32).astype(np.float64)
        pos = np.vstack([pos, 0.125 + np.float32(2.0 ** -20) * np.arange(1, 9)[:, None] * np.ones(3)])
        q = np.concatenate([q, np.full(8, 0.5)]).astype(np.float32).astype(np.float64)
    f, phi, grad = run_gpu(torch_cuda, pos, q, P, 0.5, 8, prec)
    o = oracle.FMM(pos, q, P, 0.5, 8).traverse()
    check_structure(f, o)
    assert o.counts()["depth"] >= 15
    ophi, ograd = o.evaluate()
    assert_fields(phi, ophi, grad, ograd, TOL[prec])


def test_degenerate_sizes(torch_cuda):
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    f = FMM(10, 4, 0.5, 8, "f64")
    e = torch.zeros((0, 3), dtype=torch.float64, device="cuda")
    f.build(e)
    assert f.counts()["ncell"] == 0
    phi, grad = f.evaluate(e, torch.zeros(0, dtype=torch.float64, device="cuda"))
    assert phi.numel() == 0
    p1 = torch.tensor([[0.3, 0.2, 0.1]], dtype=torch.float64, device="cuda")
    phi, grad = f.solve(p1, torch.ones(1, dtype=torch.float64, device="cuda"))
    assert phi.item() == 0 and grad.abs().max().item() == 0
    pc = torch.full((5, 3), 0.25, dtype=torch.float64, device="cuda")
    f = FMM(10, 4, 0.5, 2, "f64")          # ncrit < 5: a single-child chain to level 21 (R20)
    phi, grad = f.solve(pc, torch.ones(5, dtype=torch.float64, device="cuda"))
    assert f.counts()["depth"] == 21 and phi.abs().max().item() == 0


def test_errors(torch_cuda):
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM, FMMError
    from paper_1405_7487_b200.fmm import FMM_ERR_NONFINITE, FMM_ERR_STATE, FMM_ERR_ARG
    f = FMM(100, 4, 0.5, 8, "f64")
    p = torch.rand((10, 3), dtype=torch.float64, device="cuda")
    q = torch.rand(10, dtype=torch.float64, device="cuda")
    with pytest.raises(FMMError) as ei:
        f.evaluate(p, q)
    assert ei.value.status == FMM_ERR_STATE
    bad = p.clone()
    bad[3, 1] = float("nan")
    with pytest.raises(FMMError) as ei:
        f.build(bad)
    assert ei.value.status == FMM_ERR_NONFINITE
    with pytest.raises(FMMError) as ei:
        f.build(torch.rand((101, 3), dtype=torch.float64, device="cuda"))
    assert ei.value.status == FMM_ERR_ARG
    with pytest.raises(FMMError):
        f.build(p.float())
    f.build(p)
    with pytest.raises(FMMError) as ei:
        f.evaluate(p.clone(), q)   # not the built positions
    assert ei.value.status == FMM_ERR_STATE
    # fmm_solve: the same argument checks; NaN positions fail before any work
    with pytest.raises(FMMError) as ei:
        f.solve(torch.rand((101, 3), dtype=torch.float64, device="cuda"), torch.rand(101, dtype=torch.float64,
                                                                                      device="cuda"))
    assert ei.value.status == FMM_ERR_ARG
    with pytest.raises(FMMError) as ei:
        f.solve(bad, q)
    assert ei.value.status == FMM_ERR_NONFINITE
    from paper_1405_7487_b200.fmm import lib
    import ctypes as C
    assert lib().fmm_solve(f._h, C.c_void_p(p.data_ptr()), None, 10, C.c_void_p(q.data_ptr()),
                           C.c_void_p(q.data_ptr()), None) == FMM_ERR_ARG   # null q
    phi0, grad0 = f.solve(p[:0].contiguous(), q[:0].contiguous())   # n = 0: a no-op
    assert phi0.numel() == 0 and grad0.numel() == 0
    phi, grad = f.solve(p, q)   # and the context still works
    o = oracle.FMM(p.cpu().numpy(), q.cpu().numpy(), 4, 0.5, 8).traverse()
    assert_field(phi.cpu().numpy(), o.evaluate()[0], 1e-12)


def test_solve_host_matches_device(torch_cuda):
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    pos, q = synth.generate("plummer", 5000, 77, np.float32)
    f = FMM(5000, 6, 0.5, 32, "f32")
    phi_h, grad_h = f.solve_host(pos, q)
    phi_d, grad_d = f.solve(torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda())
    np.testing.assert_array_equal(phi_h, phi_d.cpu().numpy())
    np.testing.assert_array_equal(grad_h, grad_d.cpu().numpy())


def test_unaligned_positions_same_result(torch_cuda):
    """fp32 positions that are not 16-B aligned take the scalar gather (keys.cu), aligned ones the
    float4-pair gather: the sorted bodies, hence every output, are bit-identical."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    n = 20000
    pos, q = synth.generate("plummer", n, 93, np.float32)
    tq = torch.from_numpy(q).cuda()
    tp = torch.from_numpy(pos).cuda()
    buf = torch.empty(3 * n + 1, dtype=torch.float32, device="cuda")
    tpu = buf[1:].view(n, 3)
    tpu.copy_(tp)
    assert tp.data_ptr() % 16 == 0 and tpu.data_ptr() % 16 == 4
    f = FMM(n, 10, 0.4, 64, "f32")
    phi_a, grad_a = [t.cpu().numpy() for t in f.solve(tp, tq)]
    phi_u, grad_u = [t.cpu().numpy() for t in f.solve(tpu, tq)]
    np.testing.assert_array_equal(phi_a, phi_u)
    np.testing.assert_array_equal(grad_a, grad_u)


@pytest.mark.parametrize("prec,kind", [("f32", "cube"), ("f64", "plummer")])
def test_solve_equals_build_evaluate(torch_cuda, prec, kind, monkeypatch):
    """fmm_solve (P2M/M2M on the aux stream during the traversal, L2L/L2P during P2P, far field
    merged afterwards) gives bit-identical outputs to fmm_build + fmm_evaluate and to a context
    with every pass on the caller's stream (FMM_OVERLAP=0)."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate(kind, 30000, 91, dt)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    f = FMM(30000, 10 if prec == "f32" else 6, 0.4, 64 if prec == "f32" else 32, prec)
    phi_s, grad_s = f.solve(tp, tq)
    f.build(tp)
    phi_e, grad_e = f.evaluate(tp, tq)
    monkeypatch.setenv("FMM_OVERLAP", "0")
    g = FMM(30000, 10 if prec == "f32" else 6, 0.4, 64 if prec == "f32" else 32, prec)
    phi_0, grad_0 = g.solve(tp, tq)
    # the breadth-first traversal grouped by one radix sort of the packed pairs gives the same
    # lists (and the fields to tolerance: another M2L summation order)
    monkeypatch.setenv("FMM_DTT", "bfs")
    monkeypatch.setenv("FMM_LIST_SORT", "1")
    h = FMM(30000, 10 if prec == "f32" else 6, 0.4, 64 if prec == "f32" else 32, prec)
    phi_1, grad_1 = h.solve(tp, tq)
    torch.cuda.synchronize()
    for a, b in ((phi_s, phi_e), (grad_s, grad_e), (phi_s, phi_0), (grad_s, grad_0)):
        np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
    for a, b in zip(f.lists(), h.lists()):
        np.testing.assert_array_equal(a, b)
    for a, b in ((phi_s, phi_1), (grad_s, grad_1)):
        assert_field(a.cpu().numpy(), b.cpu().numpy(), TOL[prec])


@pytest.mark.parametrize("prec,kind,n", [("f32", "cube", 40000), ("f64", "plummer", 30000), ("f32", "sphere", 30000)])
def test_target_traversal_equals_bfs(torch_cuda, prec, kind, n, monkeypatch):
    """The target-ordered traversal (default) and the breadth-first one (FMM_DTT=bfs) give the same
    M2L and P2P lists (canonical order) and the same fields to the precision's tolerance; the
    target-ordered lists are bit-reproducible between runs."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate(kind, n, 17, dt)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    P, ncrit = (10, 64) if prec == "f32" else (6, 16)
    f = FMM(n, P, 0.4, ncrit, prec)
    phi_t, grad_t = f.solve(tp, tq)
    phi_t2, grad_t2 = f.solve(tp, tq)
    monkeypatch.setenv("FMM_DTT", "bfs")
    g = FMM(n, P, 0.4, ncrit, prec)
    phi_b, grad_b = g.solve(tp, tq)
    torch.cuda.synchronize()
    for a, b in zip(f.lists(), g.lists()):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(phi_t.cpu().numpy(), phi_t2.cpu().numpy())
    np.testing.assert_array_equal(grad_t.cpu().numpy(), grad_t2.cpu().numpy())
    tol = TOL[prec]
    assert_fields(phi_t.cpu().numpy(), phi_b.cpu().numpy(), grad_t.cpu().numpy(), grad_b.cpu().numpy(), tol)


@pytest.mark.parametrize("kind", ["plummer", "cube"])
def test_target_traversal_overflow_paths(torch_cuda, kind, monkeypatch):
    """Split lists forced over a 4-entry shared capacity (FMM_TCT_CAP=4): most targets take the
    global-memory overflow kernels, in both the count/emit and the single-pass (slot) modes; the
    lists and fields are bit-identical to the normal path."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    pos, q = synth.generate(kind, 20000, 23, np.float64)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    f = FMM(20000, 5, 0.5, 16, "f64")
    phi_a, grad_a = f.solve(tp, tq)
    monkeypatch.setenv("FMM_TCT_CAP", "4")
    monkeypatch.setenv("FMM_TCT_TIGHT", "1")   # and the sync-free pass redone after a capacity overflow
    g = FMM(20000, 5, 0.5, 16, "f64")
    for _ in range(3):   # first build: count + emit passes; then single pass into slots (sync-free)
        phi_b, grad_b = g.solve(tp, tq)
        torch.cuda.synchronize()
        for a, b in zip(f.lists(), g.lists()):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(phi_a.cpu().numpy(), phi_b.cpu().numpy())
        np.testing.assert_array_equal(grad_a.cpu().numpy(), grad_b.cpu().numpy())
    # the single pass without its overflow kernels (as after a build that had no overflowed target,
    # FMM_TCT_SKIP=1 at every level): the overflows stop it and the redo gives the same lists
    monkeypatch.delenv("FMM_TCT_TIGHT")
    monkeypatch.setenv("FMM_TCT_SKIP", "1")
    h = FMM(20000, 5, 0.5, 16, "f64")
    for _ in range(3):
        phi_c, grad_c = h.solve(tp, tq)
        torch.cuda.synchronize()
        for a, b in zip(f.lists(), h.lists()):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(phi_a.cpu().numpy(), phi_c.cpu().numpy())
        np.testing.assert_array_equal(grad_a.cpu().numpy(), grad_c.cpu().numpy())


def test_random_rebuilds_one_context(torch_cuda):
    """20 builds of random sizes and distributions on ONE context, in an order that makes the
    size-learning fast paths (tree levels, traversal slots and buffers sized from the previous
    build) meet both repeats and surprises (deeper trees, longer lists, wider levels): structure
    bit-exact and fields at tolerance every time."""
    from paper_1405_7487_b200 import FMM
    rng = np.random.default_rng(2024)
    f = FMM(16000, 4, 0.5, 16, "f64")
    for it in range(20):
        kind = ["cube", "plummer", "sphere"][int(rng.integers(3))]
        n = int(rng.integers(1, 16001)) if it % 4 else 12000   # repeats of one size too
        pos, q = synth.generate(kind, n, 100 + it if it % 4 else 7)
        tp = torch_cuda.from_numpy(pos).cuda()
        phi, grad = f.solve(tp, torch_cuda.from_numpy(q).cuda())
        o = oracle.FMM(pos, q, 4, 0.5, 16).traverse()
        check_structure(f, o)
        ophi, ograd = o.evaluate()
        assert_fields(phi.cpu().numpy(), ophi, grad.cpu().numpy(), ograd, 1e-12, f"{it} {kind} {n}")


def test_repeat_builds_reuse_context(torch_cuda):
    # ONE context across sizes and distributions: workspace growth, and the back-to-back
    # traversal sized from the previous build (smaller, larger -> overflow fallback, deeper)
    from paper_1405_7487_b200 import FMM
    f = FMM(20000, 4, 0.5, 16, "f64")
    for kind, n in (("cube", 500), ("cube", 5000), ("cube", 5000), ("cube", 800), ("plummer", 20000),
                    ("plummer", 20000), ("cube", 3000)):
        pos, q = synth.generate(kind, n, n)
        tp = torch_cuda.from_numpy(pos).cuda()
        phi, grad = f.solve(tp, torch_cuda.from_numpy(q).cuda())
        o = oracle.FMM(pos, q, 4, 0.5, 16).traverse()
        check_structure(f, o)
        ophi, ograd = o.evaluate()
        assert_fields(phi.cpu().numpy(), ophi, grad.cpu().numpy(), ograd, 1e-12)


def test_c2_full_size(torch_cuda):
    """BASELINE configs[1] at full size in the launch configuration bench.py times:
    structure bit-exact against the oracle; phi/grad on 1000 sampled targets against the
    oracle's sampled-target mode (<= 1e-5) and against the direct sum (reported)."""
    cfg = synth.CONFIGS["c2"]
    pos, q = synth.generate(cfg["kind"], cfg["n"], cfg["seed"], np.float32)
    f, phi, grad = run_gpu(torch_cuda, pos, q, cfg["P"], cfg["theta"], cfg["ncrit"], "f32")
    p64, q64 = pos.astype(np.float64), q.astype(np.float64)
    o = oracle.FMM(p64, q64, cfg["P"], cfg["theta"], cfg["ncrit"]).traverse()
    check_structure(f, o)
    t = synth.sample_targets(cfg["n"], 1000, cfg["seed"])
    ophi, ograd = o.evaluate(t)
    e_phi = oracle.rel_l2(phi[t], ophi)
    e_grad = oracle.rel_l2(grad[t], ograd)
    dphi, dgrad = oracle.direct(p64, q64, t)
    print(f"c2: vs oracle phi {e_phi:.2e} grad {e_grad:.2e}; vs direct phi {oracle.rel_l2(phi[t], dphi):.2e} "
          f"grad {oracle.rel_l2(grad[t], dgrad):.2e}")
    assert_fields(phi[t], ophi, grad[t], ograd, 1e-5, "c2")


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_root_bounds_matches_oracle(torch_cuda, prec):
    """fmm_set_root_bounds (global root cube of a Morton-range part) against the oracle built on
    the same bounds: structure bit-exact, fields at tolerance; outside bounds rejected."""
    from paper_1405_7487_b200 import FMM, FMMError
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate("plummer", 6000, 61, dt)
    b = np.array([-30.0, -20.0, -25.0, 40.0, 35.0, 30.0])
    sel = np.all((pos >= b[:3]) & (pos <= b[3:]), axis=1)
    pos, q = np.ascontiguousarray(pos[sel]), np.ascontiguousarray(q[sel])
    f = FMM(len(pos), 6, 0.5, 16, prec)
    f.set_root_bounds(b)
    tp = torch_cuda.from_numpy(pos).cuda()
    phi, grad = f.solve(tp, torch_cuda.from_numpy(q).cuda())
    o = oracle.FMM(pos.astype(np.float64), q.astype(np.float64), 6, 0.5, 16, bounds=b).traverse()
    check_structure(f, o)
    ophi, ograd = o.evaluate()
    assert_fields(phi.cpu().numpy(), ophi, grad.cpu().numpy(), ograd, TOL[prec])
    f.set_root_bounds(np.array([0.0, 0.0, 0.0, 1.0, 1.0, 1.0]))
    with pytest.raises(FMMError):
        f.build(tp)


@pytest.mark.parametrize("kind,n,ncrit", [("sphere", 30000, 512), ("plummer", 20000, 64), ("cube", 9000, 200)])
def test_mutual_p2p(torch_cuda, kind, n, ncrit, monkeypatch):
    """Mutual P2P (FMM_P2P_MUTUAL=1): each unordered leaf pair evaluated once, the
    reaction kept in per-pair slots and added in list order.  Against the oracle at the fp32
    tolerance, against the one-sided kernels (same lists, P2P summation order only), with
    coincident points (self pairs), and bit-reproducible between runs."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    pos, q = synth.generate(kind, n, 41, np.float32)
    pos[-20:] = pos[:20]                      # coincident points: r = 0 skipped in self pairs only
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    f = FMM(n, 10, 0.4, ncrit, "f32")
    phi_1, grad_1 = f.solve(tp, tq)
    monkeypatch.setenv("FMM_P2P_MUTUAL", "1")
    g = FMM(n, 10, 0.4, ncrit, "f32")
    phi_m, grad_m = g.solve(tp, tq)
    phi_m2, grad_m2 = g.solve(tp, tq)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(phi_m.cpu().numpy(), phi_m2.cpu().numpy())
    np.testing.assert_array_equal(grad_m.cpu().numpy(), grad_m2.cpu().numpy())
    pm, gm = phi_m.cpu().numpy().astype(np.float64), grad_m.cpu().numpy().astype(np.float64)
    assert_fields(pm, phi_1.cpu().numpy(), gm, grad_1.cpu().numpy(), TOL["f32"])
    o = oracle.FMM(pos.astype(np.float64), q.astype(np.float64), 10, 0.4, ncrit).traverse()
    t = synth.sample_targets(n, 400, 41)
    ophi, ograd = o.evaluate(t)
    assert_fields(pm[t], ophi, gm[t], ograd, TOL["f32"])


SWITCHES = [
    # every FMM_* alternative the library keeps (DESIGN.md §5 "Switches"), against the oracle
    ({"FMM_P2P_VARIANT": "1"}, "f32"),                    # k_p2p_f32: a warp per target leaf
    ({"FMM_P2P_GENERIC": "1"}, "f32"),                    # k_p2p_generic<float>
    ({"FMM_M2L_GENERIC": "1"}, "f32"),                    # generic M2L (m2l.cu) in fp32
    ({"FMM_M2L_VARIANT": "1"}, "f32"),                    # scalar register M2L k_m2l_fast<10, float>
    ({"FMM_P2P_MUTUAL": "2"}, "f32"),                     # mutual P2P only for big leaves
    ({"FMM_PRIO": "0"}, "f32"),                           # no high-priority critical-path stream
    ({"FMM_TREE_FAST": "0"}, "f64"),                      # one host round trip per tree level
    ({"FMM_TCT_SINGLE": "0"}, "f64"),                     # count + emit traversal every build
    ({"FMM_DTT": "bfs", "FMM_CANONICAL_M2L": "0"}, "f32"),
    ({"FMM_DTT": "bfs", "FMM_LIST_SORT": "1"}, "f64"),
    ({"FMM_OVERLAP": "0", "FMM_P2P_GENERIC": "1", "FMM_M2L_GENERIC": "1"}, "f64"),
    # the staged onesweep pass (default only above one wave of tiles) for the Morton pairs and,
    # through the breadth-first lists, the keys-only sort
    ({"FMM_SORT_STAGED": "1", "FMM_DTT": "bfs", "FMM_LIST_SORT": "1"}, "f32"),
]


@pytest.mark.parametrize("env,prec", SWITCHES, ids=[",".join(f"{k}={v}" for k, v in e.items()) for e, _ in SWITCHES])
def test_switch_alternatives(torch_cuda, env, prec, monkeypatch):
    """Each default-off alternative kernel or schedule: structure bit-exact and fields within the
    precision's tolerance against the oracle, on two builds of one context (first build and the
    size-learning rebuild), Plummer (adaptive, tiny and huge leaves) at P = 10 in fp32, P = 6 fp64."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    dt = np.float32 if prec == "f32" else np.float64
    P, ncrit = (10, 64) if prec == "f32" else (6, 16)
    for kind, n, seed in (("plummer", 20000, 131), ("cube", 12000, 132)):
        pos, q = synth.generate(kind, n, seed, dt)
        f = FMM(n, P, 0.4, ncrit, prec)
        tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
        f.solve(tp, tq)
        phi, grad = f.solve(tp, tq)
        torch.cuda.synchronize()
        o = oracle.FMM(pos.astype(np.float64), q.astype(np.float64), P, 0.4, ncrit).traverse()
        check_structure(f, o)
        ophi, ograd = o.evaluate()
        assert_fields(phi.cpu().numpy(), ophi, grad.cpu().numpy(), ograd, TOL[prec], f"{env} {kind}")


@pytest.mark.parametrize("kind,n,P,theta,ncrit,prec", [("cube", 4096, 4, 0.5, 32, "f64"),
                                                       ("plummer", 5000, 10, 0.4, 64, "f32"),
                                                       ("sphere", 3000, 6, 0.5, 16, "f64")])
def test_debug_stages_on_oracle_tree(torch_cuda, kind, n, P, theta, ncrit, prec):
    """fmm_debug_p2p / fmm_debug_m2l (SURVEY §8(b) debug entry points) fed the ORACLE's sorted
    bodies, cells and canonical lists: the product P2P kernels against per-pair oracle.p2p (R17)
    sums, the product M2L kernels against per-pair oracle.m2l (R14) sums on the oracle's M."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    dt = np.float32 if prec == "f32" else np.float64
    tdt = torch.float32 if prec == "f32" else torch.float64
    pos, q = synth.generate(kind, n, 300 + n, dt)
    p64, q64 = pos.astype(np.float64), q.astype(np.float64)
    o = oracle.FMM(p64, q64, P, theta, ncrit).traverse()
    o.evaluate()
    _, perm = o.sorted()
    cells = o.cells()
    m2l, p2p = o.lists()
    M, _ = o.expansions()
    sp, sq = p64[perm], q64[perm]
    bb, bc = cells["body_begin"], cells["body_count"]
    # references: per-pair sums of the pinned oracle stage functions
    rphi = np.zeros(n); rgrad = np.zeros((n, 3))
    for a, b in p2p:
        ph, gr = oracle.p2p(sp[bb[a]:bb[a] + bc[a]], sp[bb[b]:bb[b] + bc[b]], sq[bb[b]:bb[b] + bc[b]])
        rphi[bb[a]:bb[a] + bc[a]] += ph
        rgrad[bb[a]:bb[a] + bc[a]] += gr
    rL = np.zeros_like(M)
    c = cells["center"]
    for a, b in m2l:
        oracle.m2l(P, M[b], c[a] - c[b], rL[a])
    f = FMM(n, P, theta, ncrit, prec)
    cu = lambda x, d=None: torch.from_numpy(np.ascontiguousarray(x if d is None else x.astype(d))).cuda()  # noqa: E731
    u32 = lambda x: cu(x.astype(np.int32))  # noqa: E731
    phi, grad = f.debug_p2p(cu(pos[perm]), cu(q[perm]), u32(bb), u32(bc), u32(cells["child_count"]), u32(p2p))
    torch.cuda.synchronize()
    assert phi.dtype == tdt
    assert_fields(phi.cpu().numpy(), rphi, grad.cpu().numpy(), rgrad, TOL[prec], "debug_p2p")
    h = 0.5 * float(np.max(cells["bmax"][0] - cells["bmin"][0]))   # R2 half-width (root box = all bodies)
    L = f.debug_m2l(cu(c), cu(cells["level"]), cu(M), h, u32(m2l)).cpu().numpy()
    # fp64 kernels: 1e-11 of the largest coefficient; fp32 M2L arithmetic (R19): per degree, the
    # fp32 operand rounding relative to that degree's largest coefficient
    tol = 1e-11 if prec == "f64" else 2e-5
    ex = oracle.multi_indices(P).sum(axis=1)
    for deg in range(P):
        k = ex == deg
        scale = np.abs(rL[:, k]).max()
        assert np.abs(L[:, k] - rL[:, k]).max() <= tol * scale, (deg, np.abs(L[:, k] - rL[:, k]).max() / scale)
    # a list out of canonical order is rejected
    from paper_1405_7487_b200 import FMMError
    bad = p2p[::-1].copy()
    with pytest.raises(FMMError):
        f.debug_p2p(cu(pos[perm]), cu(q[perm]), u32(bb), u32(bc), u32(cells["child_count"]), u32(bad))
