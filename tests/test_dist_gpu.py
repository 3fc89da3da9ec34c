"""Multi-GPU path on ONE GPU: K ranks of the library's distributed driver
(fmm_create_dist + fmm_dist_solve, csrc/dist.cu) in one process -- an in-process group (fmm_group),
one host thread per rank -- checked against the oracle's per-partition mode
(oracle.traverse_pair / evaluate_multi).

Bar: rank i's lists over (local tree + grafted LETs) equal the oracle's
lists of T_i against every full local tree S_j, bit-exact (remote sources mapped back to the
sender's cell ids); phi / grad against evaluate_multi at the §8(c) tolerances.  The ranks
meet at host barriers; no kernel waits on another rank's kernel.
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


class Ranks:
    """K DistFMM contexts of one LocalGroup and their last step's results."""

    def __init__(self, torch, K, n_max, P, theta, ncrit, prec, part="morton"):
        from paper_1405_7487_b200.dist import DistFMM, LocalGroup
        self.torch, self.K = torch, K
        self.group = LocalGroup(K)
        self.fmm = [DistFMM(n_max, P, theta, ncrit, prec, 0, K, r, group=self.group, partitioner=part)
                    for r in range(K)]
        self.streams = [torch.cuda.Stream() for _ in range(K)]

    def solve(self, P_in, Q_in, bases, reuse_weights=False):
        from paper_1405_7487_b200.dist import run_ranks

        def body(r):
            st = self.streams[r]
            out = self.fmm[r].solve(P_in[r], Q_in[r], bases[r], reuse_weights=reuse_weights, stream=st)
            st.synchronize()
            return out
        out = run_ranks(body, self.K)
        self.local = [f.local() for f in self.fmm]             # (gids, peers) per rank
        return out

    @property
    def global_bounds(self):
        return self.fmm[0].stats()["bounds"]

    def close(self):
        for f in self.fmm:
            f.close()
        self.group.close()


def split_input(torch, pos, q, K):
    # initial ownership: contiguous index slices (not spatial), as a user would hold them
    n = len(pos)
    cuts = np.linspace(0, n, K + 1).astype(int)
    P_in = [torch.from_numpy(np.ascontiguousarray(pos[cuts[r]:cuts[r + 1]])).cuda() for r in range(K)]
    Q_in = [torch.from_numpy(np.ascontiguousarray(q[cuts[r]:cuts[r + 1]])).cuda() for r in range(K)]
    return P_in, Q_in, [int(c) for c in cuts[:-1]]


def run_dist(torch, kind, n, K, P, theta, ncrit, prec, seed, part="morton"):
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate(kind, n, seed, dt)
    P_in, Q_in, bases = split_input(torch, pos, q, K)
    D = Ranks(torch, K, n, P, theta, ncrit, prec, part)
    out = D.solve(P_in, Q_in, bases)
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
    gids = [g for g, _ in D.local]
    # every particle lands on exactly one rank, and the ranks are Morton ranges of similar size
    allg = np.sort(np.concatenate(gids))
    np.testing.assert_array_equal(allg, np.arange(n))
    sizes = np.array([len(g) for g in gids])
    assert sizes.min() >= 0.5 * n / K, sizes
    if part == "orb":   # ORB boxes are axis-aligned and disjoint: each rank's particles lie in its box
        from oracle import keys as okeys
        k = okeys(pos.astype(np.float64))
        boxes = D.fmm[0].orb_boxes()
        for r in range(K):
            assert np.array_equal(D.fmm[r].orb_boxes(), boxes)      # every rank made the same plan
            kk = k[gids[r]]
            for a in range(3):
                c = np.zeros(len(kk), dtype=np.int64)
                for l in range(21):
                    c |= (((kk >> np.uint64(3 * l + a)) & np.uint64(1)).astype(np.int64)) << l
                assert np.all((c >= boxes[r, a]) & (c < boxes[r, 3 + a]))
    # oracle trees of every rank, built from the rank's particles in the order the rank holds them
    rb = D.global_bounds if part == "morton" else None   # the root cube the ranks built on
    O = [oracle.FMM(pos[g].astype(np.float64), q[g].astype(np.float64), P, theta, ncrit, bounds=rb) for g in gids]
    for i in range(K):
        f = D.fmm[i]
        m2l, p2p = f.lists()
        nci = f.counts()["ncell"]
        peers = D.local[i][1]
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
    st = [f.stats() for f in D.fmm]
    assert all(np.array_equal(x["bounds"], st[0]["bounds"]) for x in st)
    assert sum(x["n_local"] for x in st) == n
    for i in range(K):
        o_phi, o_grad = oracle.evaluate_multi(O[i], [O[j] for j in range(K) if j != i])
        ref_phi[gids[i]] = o_phi
        ref_grad[gids[i]] = o_grad
    assert_fields(phi, ref_phi, grad, ref_grad, TOL[prec], f"{kind} K={K} {part}")
    # and the whole-system FMM is an approximation of the direct sum
    t = synth.sample_targets(n, 200, 7)
    dp, dg = oracle.direct(pos.astype(np.float64), q.astype(np.float64), t)
    assert oracle.rel_l2(phi[t], dp) <= 1e-2 and oracle.rel_l2(grad[t], dg) <= 5e-2
    D.close()


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
        for k, j in enumerate(D.local[i][1]):
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
    for k, j in enumerate(D.local[i][1]):
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
    torch = torch_cuda
    n, K = 20000, 4
    pos, q = synth.generate("plummer", n, 77, np.float64)
    P_in, Q_in, bases = split_input(torch, pos, q, K)
    D = Ranks(torch, K, n, 4, 0.5, 16, "f64")
    D.solve(P_in, Q_in, bases)
    w1 = np.concatenate([D.fmm[r].weights(len(P_in[r])) for r in range(K)]).astype(np.float64)  # owner order
    g1 = [g for g, _ in D.local]
    share1 = np.array([w1[g].sum() for g in g1]) / w1.sum()
    D.solve(P_in, Q_in, bases, reuse_weights=True)
    g2 = [g for g, _ in D.local]
    share2 = np.array([w1[g].sum() for g in g2]) / w1.sum()
    assert np.abs(share2 - 1.0 / K).max() < 0.01, share2
    assert np.abs(share1 - 1.0 / K).max() > np.abs(share2 - 1.0 / K).max(), (share1, share2)
    # the same weights given explicitly (fmm_set_weights) make the same partition
    for r in range(K):
        D.fmm[r].set_weights(torch.from_numpy(w1[bases[r]:bases[r] + len(P_in[r])].astype(np.float32)).cuda())
    D.solve(P_in, Q_in, bases)
    for a, b in zip(g2, [g for g, _ in D.local]):
        np.testing.assert_array_equal(a, b)
    D.close()


@pytest.mark.parametrize("part", ["morton", "orb"])
def test_dist_degenerate(torch_cuda, part):
    """Ranks left empty by the partition (3 particles on 4 ranks; all particles coincident):
    the distributed path still returns the direct sum."""
    torch = torch_cuda
    for pos in (np.array([[0.1, 0.2, 0.3], [0.9, 0.8, 0.7], [0.5, 0.5, 0.1]]),
                np.tile(np.array([[0.25, 0.5, 0.75]]), (40, 1))):
        n, K = len(pos), 4
        q = np.linspace(-1.0, 1.0, n)
        P_in, Q_in, bases = split_input(torch, pos, q, K)
        D = Ranks(torch, K, n, 4, 0.5, 2, "f64", part)
        out = D.solve(P_in, Q_in, bases)
        phi = np.concatenate([o[0].cpu().numpy() for o in out])
        grad = np.concatenate([o[1].cpu().numpy() for o in out])
        dp, dg = oracle.direct(pos, q)
        np.testing.assert_allclose(phi, dp, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(grad, dg, rtol=1e-12, atol=1e-12)
        D.close()


def test_alpha_tuning_steps(torch_cuda):
    """Eq. (1) alpha optimised over time steps (fmm_dist_tune_alpha): a tuned
    multi-step run changes alpha between steps (probes of the golden-section search), every rank
    uses the same alpha, and every step still returns the direct sum within the FMM error of a
    single-rank solve."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    n, K = 12000, 3
    pos, q = synth.generate("plummer", n, 5, np.float64)
    P_in, Q_in, bases = split_input(torch, pos, q, K)
    D = Ranks(torch, K, n, 6, 0.5, 16, "f64")
    for f in D.fmm:
        f.tune_alpha(0.25, 4.0, 0.2)
    t = synth.sample_targets(n, 300, 5)
    dphi, dgrad = oracle.direct(pos, q, t)
    f1 = FMM(n, 6, 0.5, 16, "f64")
    p1, _ = f1.solve(torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda())
    e1 = oracle.rel_l2(p1.cpu().numpy()[t], dphi)
    alphas = []
    for _ in range(8):
        out = D.solve(P_in, Q_in, bases, reuse_weights=True)
        al = [f.alpha for f in D.fmm]
        assert len(set(al)) == 1, al
        alphas.append(al[0])
        phi = np.concatenate([o[0].cpu().numpy() for o in out])
        grad = np.concatenate([o[1].cpu().numpy() for o in out])
        assert oracle.rel_l2(phi[t], dphi) < 10 * e1 + 1e-12
        assert oracle.rel_l2(grad[t], dgrad) < 1e-3
    assert len(set(alphas)) >= 2, alphas
    assert D.fmm[0].stats()["tuner_probes"] >= 3
    D.close()


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_partition_overlap_bit_identical(torch_cuda, prec, monkeypatch):
    """f1: the staying particles sorted while the partition exchange flies and the
    arrivals merged in (default) give bit-identical keys, permutation, cells, lists and fields to a
    full sort after the exchange (FMM_DIST_SORT=0), over two steps with reused Eq. (1) weights."""
    torch = torch_cuda
    n, K = 30000, 3
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate("plummer", n, 12, dt)
    P_in, Q_in, bases = split_input(torch, pos, q, K)
    A = Ranks(torch, K, n, 6, 0.5, 32, prec)
    monkeypatch.setenv("FMM_DIST_SORT", "0")
    B = Ranks(torch, K, n, 6, 0.5, 32, prec)
    for reuse in (False, True):
        oa = A.solve(P_in, Q_in, bases, reuse_weights=reuse)
        ob = B.solve(P_in, Q_in, bases, reuse_weights=reuse)
        for r in range(K):
            np.testing.assert_array_equal(oa[r][0].cpu().numpy(), ob[r][0].cpu().numpy())
            np.testing.assert_array_equal(oa[r][1].cpu().numpy(), ob[r][1].cpu().numpy())
            fa, fb = A.fmm[r], B.fmm[r]
            for x, y in zip(fa.sorted(), fb.sorted()):
                np.testing.assert_array_equal(x, y)
            for x, y in zip(fa.lists(), fb.lists()):
                np.testing.assert_array_equal(x, y)
    A.close()
    B.close()


@pytest.mark.parametrize("split", ["0", "1"])
def test_dist_timeline_overlap(torch_cuda, split, monkeypatch):
    """fmm_dist_timeline: the LET structure exchange is posted before the local traversal (their
    spans overlap or the exchange ends first), the data exchange starts after the upward pass, and
    the staying-particle sort starts before the particle exchange ends; with FMM_DIST_SPLIT=1 the
    local interactions start before the remote fragments are traversed."""
    torch = torch_cuda
    monkeypatch.setenv("FMM_DIST_SPLIT", split)
    n, K = 60000, 2
    pos, q = synth.generate("cube", n, 3, np.float32)
    P_in, Q_in, bases = split_input(torch, pos, q, K)
    D = Ranks(torch, K, n, 10, 0.4, 64, "f32")
    for f in D.fmm:
        f.set_timing(True)
    D.solve(P_in, Q_in, bases)
    D.solve(P_in, Q_in, bases, reuse_weights=True)
    for f in D.fmm:
        tl = f.timeline()
        assert tl["let_struct_exchange"][0] <= tl["local_dtt"][0] + 1e-3, tl
        assert tl["let_data_exchange"][1] >= tl["upward"][1] - 1e-3, tl
        assert tl["stay_sort"][0] <= tl["particle_exchange"][1] + 1e-3, tl
        if split == "1":   # split interactions: the local M2L/P2P start before the remote traversal
            assert 0 <= tl["interact_local"][0] <= tl["remote_dtt"][0] + 1e-3, tl
            assert tl["interact_remote"][0] >= tl["interact_local"][0], tl
    D.close()


@pytest.mark.parametrize("prec,part", [("f32", "morton"), ("f64", "orb")])
def test_split_interactions_match_unsplit(torch_cuda, prec, part, monkeypatch):
    """Local M2L/P2P launched right after the local traversal and the remote lists' interactions
    added after the fragments (FMM_DIST_SPLIT=1) against one pass over the concatenated lists
    (default), over 6 steps with reused Eq. (1) weights (buffer rotations between steps): the same
    lists bit for bit, the same fields to the precision's tolerance (only the summation order
    differs)."""
    torch = torch_cuda
    n, K = 24000, 3
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate("plummer", n, 19, dt)
    P_in, Q_in, bases = split_input(torch, pos, q, K)
    P, ncrit = (10, 64) if prec == "f32" else (6, 16)
    monkeypatch.setenv("FMM_DIST_SPLIT", "1")
    A = Ranks(torch, K, n, P, 0.4, ncrit, prec, part)
    monkeypatch.setenv("FMM_DIST_SPLIT", "0")
    B = Ranks(torch, K, n, P, 0.4, ncrit, prec, part)
    for step in range(6):
        oa = A.solve(P_in, Q_in, bases, reuse_weights=True)
        ob = B.solve(P_in, Q_in, bases, reuse_weights=True)
        for r in range(K):
            for x, y in zip(A.fmm[r].lists(), B.fmm[r].lists()):
                np.testing.assert_array_equal(x, y)
            assert A.fmm[r].counts() == B.fmm[r].counts()
        phi_a = np.concatenate([o[0].cpu().numpy() for o in oa]); phi_b = np.concatenate([o[0].cpu().numpy() for o in ob])
        grad_a = np.concatenate([o[1].cpu().numpy() for o in oa]); grad_b = np.concatenate([o[1].cpu().numpy() for o in ob])
        assert_fields(phi_a, phi_b, grad_a, grad_b, TOL[prec], f"split vs unsplit, step {step}")
    A.close()
    B.close()


def test_nccl_transport_single_rank(torch_cuda):
    """The NCCL transport (libnccl dlopen'ed by the library, communicator from a unique id) with one
    rank: fmm_dist_solve returns the single-GPU result bit for bit, twice (the second step with the
    Eq. (1) weights of the first)."""
    torch = torch_cuda
    from paper_1405_7487_b200 import FMM
    from paper_1405_7487_b200.dist import DistFMM, nccl_unique_id
    pos, q = synth.generate("plummer", 20000, 13, np.float32)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    D = DistFMM(20000, 10, 0.4, 64, "f32", 0, 1, 0, unique_id=nccl_unique_id())
    f = FMM(20000, 10, 0.4, 64, "f32")
    p1, g1 = f.solve(tp, tq)
    for reuse in (False, True):
        p, g = D.solve(tp, tq, 0, reuse_weights=reuse)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(p.cpu().numpy(), p1.cpu().numpy())
        np.testing.assert_array_equal(g.cpu().numpy(), g1.cpu().numpy())
    assert D.stats()["n_local"] == 20000 and D.stats()["npeers"] == 0
    D.close()
