"""Multi-GPU path on ONE GPU: K ranks driven by one process (LoopbackComm),
checked against the oracle's per-partition mode (oracle.traverse_pair / evaluate_multi).

Bar: rank i's lists over (local tree + grafted LETs) equal the oracle's
lists of T_i against every full local tree S_j, bit-exact (remote sources mapped back to the
sender's cell ids); phi / grad against evaluate_multi at the §8(c) tolerances.  The ranks
run one after another: no kernel waits on another rank's kernel.
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


def run_dist(torch, kind, n, K, P, theta, ncrit, prec, seed, part="morton"):
    from paper_1405_7487_b200.dist import DistFMM, LoopbackComm
    dt = np.float32 if prec == "f32" else np.float64
    tdt = torch.float32 if prec == "f32" else torch.float64
    pos, q = synth.generate(kind, n, seed, dt)
    # initial ownership: contiguous index slices (not spatial), as a user would hold them
    cuts = np.linspace(0, n, K + 1).astype(int)
    P_in = [torch.from_numpy(pos[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    Q_in = [torch.from_numpy(q[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    D = DistFMM(LoopbackComm(K), n, P, theta, ncrit, prec, partitioner=part)
    out = D.solve(P_in, Q_in, [int(c) for c in cuts[:-1]])
    torch.cuda.synchronize()
    phi = np.concatenate([o[0].cpu().numpy() for o in out]).astype(np.float64)
    grad = np.concatenate([o[1].cpu().numpy() for o in out]).astype(np.float64)
    return D, pos, q, phi, grad


CASES = [
    # kind, n, K, P, theta, ncrit, prec, partitioner
    ("cube", 6000, 2, 4, 0.5, 32, "f64", "morton"),
    ("cube", 9000, 3, 6, 0.4, 16, "f64", "morton"),
    ("plummer", 8000, 4, 5, 0.5, 16, "f64", "morton"),
    ("cube", 20000, 4, 10, 0.4, 64, "f32", "morton"),
    ("plummer", 12000, 3, 10, 0.4, 64, "f32", "morton"),
    ("sphere", 5000, 2, 4, 0.6, 8, "f32", "morton"),
    # ORB multisection, including non-power-of-two rank counts
    ("cube", 9000, 3, 6, 0.4, 16, "f64", "orb"),
    ("plummer", 12000, 5, 10, 0.4, 64, "f32", "orb"),
    ("sphere", 6000, 4, 4, 0.6, 8, "f64", "orb"),
]


@pytest.mark.parametrize("kind,n,K,P,theta,ncrit,prec,part", CASES)
def test_dist_lists_and_fields(torch_cuda, kind, n, K, P, theta, ncrit, prec, part):
    D, pos, q, phi, grad = run_dist(torch_cuda, kind, n, K, P, theta, ncrit, prec, 500 + n + K, part)
    lpos, lq, lgid = D.local
    gids = [g.cpu().numpy() for g in lgid]
    # every particle lands on exactly one rank, and the ranks are Morton ranges of similar size
    allg = np.sort(np.concatenate(gids))
    np.testing.assert_array_equal(allg, np.arange(n))
    sizes = np.array([len(g) for g in gids])
    assert sizes.min() >= 0.5 * n / K, sizes
    if part == "orb":   # ORB boxes are axis-aligned and disjoint: each rank's particles lie in its box
        from oracle import keys as okeys
        k = okeys(pos.astype(np.float64))
        for r, g in D.orb_groups.items():
            kk = k[gids[r]]
            for a in range(3):
                c = np.zeros(len(kk), dtype=np.int64)
                for l in range(21):
                    c |= (((kk >> np.uint64(3 * l + a)) & np.uint64(1)).astype(np.int64)) << l
                assert np.all((c >= g["lo"][a]) & (c < g["hi"][a]))
    # oracle trees of every rank, built from the rank's particles in the order the rank holds them
    rb = D.global_bounds if part == "morton" else None   # the root cube the ranks built on
    O = [oracle.FMM(pos[g].astype(np.float64), q[g].astype(np.float64), P, theta, ncrit, bounds=rb) for g in gids]
    for i in range(K):
        f = D.fmm[i]
        m2l, p2p = f.lists()
        nci = f.counts()["ncell"]
        peers = D._peers[i]
        regions = [f.let_remote(k) for k in range(len(peers))]

        def split(lst):
            loc = lst[lst[:, 1] < nci]
            rem = {}
            for k, j in enumerate(peers):
                base, ncl, _, orig = regions[k]
                sel = (lst[:, 1] >= base) & (lst[:, 1] < base + ncl)
                r = lst[sel].copy()
                r[:, 1] = orig[r[:, 1] - base]
                rem[j] = r
            assert len(loc) + sum(len(r) for r in rem.values()) == len(lst)
            return loc, rem

        lm, rm = split(m2l)
        lp_, rp = split(p2p)
        om, op = O[i].traverse().lists()
        np.testing.assert_array_equal(lm, om)
        np.testing.assert_array_equal(lp_, op)
        for j in range(K):
            if j == i:
                continue
            tm, tp = oracle.traverse_pair(O[i], O[j])
            gm = rm.get(j, np.zeros((0, 2), np.uint32))
            gp = rp.get(j, np.zeros((0, 2), np.uint32))
            np.testing.assert_array_equal(gm, tm, err_msg=f"M2L rank {i} <- {j}")
            np.testing.assert_array_equal(gp, tp, err_msg=f"P2P rank {i} <- {j}")
    # fields: rank-local results against the oracle's multi-tree evaluation, and the gathered
    # (original-order) results against the same numbers
    ref_phi = np.zeros(n); ref_grad = np.zeros((n, 3))
    for i in range(K):
        o_phi, o_grad = oracle.evaluate_multi(O[i], [O[j] for j in range(K) if j != i])
        ref_phi[gids[i]] = o_phi
        ref_grad[gids[i]] = o_grad
    assert_fields(phi, ref_phi, grad, ref_grad, TOL[prec], f"{kind} K={K} {part}")
    # and the whole-system FMM is an approximation of the direct sum
    t = synth.sample_targets(n, 200, 7)
    dp, dg = oracle.direct(pos.astype(np.float64), q.astype(np.float64), t)
    assert oracle.rel_l2(phi[t], dp) <= 1e-2 and oracle.rel_l2(grad[t], dg) <= 5e-2


def test_dist_single_rank_equals_single_gpu(torch_cuda):
    """K = 1: partition + LET machinery reduce to the single-GPU path, bit for bit."""
    import torch
    from paper_1405_7487_b200 import FMM
    D, pos, q, phi, grad = run_dist(torch, "cube", 5000, 1, 6, 0.5, 32, "f64", 11)
    f = FMM(5000, 6, 0.5, 32, "f64")
    p1, g1 = f.solve(torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda())
    np.testing.assert_array_equal(phi, p1.cpu().numpy())
    np.testing.assert_array_equal(grad, g1.cpu().numpy())


def test_let_needs_subset_of_remote_tree(torch_cuda):
    """The LET a rank receives is a strict subset of the sender's tree (far cells are cut)."""
    D, pos, q, phi, grad = run_dist(torch_cuda, "cube", 30000, 4, 4, 0.5, 16, "f64", 21)
    for i in range(4):
        f = D.fmm[i]
        for k, j in enumerate(D._peers[i]):
            _, ncl, nbd, orig = f.let_remote(k)
            assert ncl < D.fmm[j].counts()["ncell"]
            assert nbd < D.fmm[j].counts()["n"]
            assert np.all(np.diff(orig.astype(np.int64)) > 0)   # sender order kept


def _host_work(D, i, c, alpha):
    """Eq. (1) weights of rank i recomputed on the host from its lists and cells."""
    f = D.fmm[i]
    cells = f.cells()
    nci = len(cells["level"])
    bc = cells["body_count"].astype(np.float64)
    m2l, p2p = f.lists()
    # body counts of every source index (local cells, then each grafted LET)
    src_bc = {}
    for k, j in enumerate(D._peers[i]):
        base, ncl, _, orig = f.let_remote(k)
        rb = D.fmm[j].cells()["body_count"].astype(np.float64)[orig]
        for t in range(ncl):
            src_bc[base + t] = rb[t]
    def bcount(s):
        return bc[s] if s < nci else src_bc[s]
    ml = np.zeros(nci); mr = np.zeros(nci)
    for a, b in m2l:
        if b < nci:
            ml[a] += c / bc[a]
        else:
            mr[a] += c / bc[a]
    pl = np.zeros(nci); pr = np.zeros(nci)
    for a, b in p2p:
        if b < nci:
            pl[a] += bcount(b)
        else:
            pr[a] += bcount(b)
    _, perm = f.sorted()
    w = np.zeros(f.counts()["n"])
    for a in np.nonzero(cells["child_count"] == 0)[0]:
        l, r = pl[a], pr[a]
        x = a
        while x >= 0:
            l += ml[x]; r += mr[x]
            x = cells["parent"][x]
        b0, m = cells["body_begin"][a], cells["body_count"][a]
        w[perm[b0:b0 + m]] = l + alpha * r
    return w


@pytest.mark.parametrize("K", [1, 3])
def test_work_weights_eq1(torch_cuda, K):
    """fmm_work (Eq. (1)) against the same weights recomputed from the lists."""
    D, pos, q, phi, grad = run_dist(torch_cuda, "plummer", 6000, K, 4, 0.5, 16, "f64", 41 + K)
    for i in range(K):
        c, alpha = 37.5, 0.25
        w, lr = D.fmm[i].work(c, alpha)
        ref = _host_work(D, i, c, alpha)
        np.testing.assert_allclose(w.cpu().numpy(), ref, rtol=2e-6)
        if K == 1:
            assert lr[1] == 0.0   # no remote sources on one rank


def test_weighted_partition_balances_work(torch_cuda):
    """Second step partitions with the first step's Eq. (1) weights: the ranks' shares of the
    (first-step) work are balanced, where the unweighted split by particle count is not."""
    import torch
    from paper_1405_7487_b200.dist import DistFMM, LoopbackComm
    n, K = 20000, 4
    pos, q = synth.generate("plummer", n, 77, np.float64)
    cuts = np.linspace(0, n, K + 1).astype(int)
    P_in = [torch.from_numpy(pos[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    Q_in = [torch.from_numpy(q[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    D = DistFMM(LoopbackComm(K), n, 4, 0.5, 16, "f64")
    D.solve(P_in, Q_in, [int(c) for c in cuts[:-1]])
    w1 = np.concatenate([w.cpu().numpy() for w in D.weights]).astype(np.float64)   # owner order = global order
    g1 = [g.cpu().numpy() for g in D.local[2]]
    share1 = np.array([w1[g].sum() for g in g1]) / w1.sum()
    D.solve(P_in, Q_in, [int(c) for c in cuts[:-1]], reuse_weights=True)
    g2 = [g.cpu().numpy() for g in D.local[2]]
    share2 = np.array([w1[g].sum() for g in g2]) / w1.sum()
    assert np.abs(share2 - 1.0 / K).max() < 0.01, share2
    assert np.abs(share1 - 1.0 / K).max() > np.abs(share2 - 1.0 / K).max(), (share1, share2)


@pytest.mark.parametrize("part", ["morton", "orb"])
def test_dist_degenerate(torch_cuda, part):
    """Ranks left empty by the partition (3 particles on 4 ranks; all particles coincident):
    the distributed path still returns the direct sum."""
    import torch
    from paper_1405_7487_b200.dist import DistFMM, LoopbackComm
    for pos in (np.array([[0.1, 0.2, 0.3], [0.9, 0.8, 0.7], [0.5, 0.5, 0.1]]),
                np.tile(np.array([[0.25, 0.5, 0.75]]), (40, 1))):
        n, K = len(pos), 4
        q = np.linspace(-1.0, 1.0, n)
        cuts = np.linspace(0, n, K + 1).astype(int)
        P_in = [torch.from_numpy(np.ascontiguousarray(pos[cuts[r]:cuts[r + 1]])).cuda() for r in range(K)]
        Q_in = [torch.from_numpy(np.ascontiguousarray(q[cuts[r]:cuts[r + 1]])).cuda() for r in range(K)]
        D = DistFMM(LoopbackComm(K), n, 4, 0.5, 2, "f64", partitioner=part)
        out = D.solve(P_in, Q_in, [int(c) for c in cuts[:-1]])
        phi = np.concatenate([o[0].cpu().numpy() for o in out])
        grad = np.concatenate([o[1].cpu().numpy() for o in out])
        dp, dg = oracle.direct(pos, q)
        np.testing.assert_allclose(phi, dp, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(grad, dg, rtol=1e-12, atol=1e-12)
        D.close()


def test_alpha_tuning_steps(torch_cuda):
    """Eq. (1) alpha optimised over time steps: a tuned multi-step run changes
    alpha between steps (probes of the golden-section search), and every step still returns the
    direct sum within the FMM error of a single-rank solve."""
    import torch
    from paper_1405_7487_b200 import FMM
    from paper_1405_7487_b200.dist import DistFMM, LoopbackComm
    n, K = 12000, 3
    pos, q = synth.generate("plummer", n, 5, np.float64)
    cuts = np.linspace(0, n, K + 1).astype(int)
    P_in = [torch.from_numpy(pos[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    Q_in = [torch.from_numpy(q[cuts[r]:cuts[r + 1]]).cuda() for r in range(K)]
    D = DistFMM(LoopbackComm(K), n, 6, 0.5, 16, "f64")
    tu = D.enable_alpha_tuning(lo=0.25, hi=4.0, tol=0.2)
    t = synth.sample_targets(n, 300, 5)
    dphi, dgrad = oracle.direct(pos, q, t)
    f1 = FMM(n, 6, 0.5, 16, "f64")
    p1, _ = f1.solve(torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda())
    e1 = oracle.rel_l2(p1.cpu().numpy()[t], dphi)
    alphas = []
    for _ in range(8):
        out = D.solve(P_in, Q_in, [int(c) for c in cuts[:-1]], reuse_weights=True)
        alphas.append(D.alpha)
        phi = np.concatenate([o[0].cpu().numpy() for o in out])
        grad = np.concatenate([o[1].cpu().numpy() for o in out])
        assert oracle.rel_l2(phi[t], dphi) < 10 * e1 + 1e-12
        assert oracle.rel_l2(grad[t], dgrad) < 1e-3
    assert len(set(alphas)) >= 2, alphas
    assert len(tu.history) >= 3
    D.close()
