"""Pins of the CPU oracle against what the paper and the mathematics fix (CPU only).

Each test names the rule and the independent fact
it checks: closed forms, exact identities of the Cartesian basis, harmonicity of 1/r,
finite differences, brute force on tiny inputs, the direct sum, truncation-error decay
O(theta^P) (§III-A) and the momentum invariant (north_star).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


# ---------------------------------------------------------------- R1 / R17 --
def test_p2p_closed_forms(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "closed_forms.json")))
    for case in g["p2p"]:
        phi, grad = oracle.p2p([case["target"]], [case["source"]], [case["q"]])
        assert phi[0] == case["phi"], case["what"]
        np.testing.assert_array_equal(grad[0], case["grad"])


def test_direct_two_unit_charges():
    # two unit charges at distance 1 -> each potential 1
    phi, grad = oracle.direct([[0, 0, 0], [0, 1, 0]], [1.0, 1.0])
    np.testing.assert_array_equal(phi, [1.0, 1.0])
    np.testing.assert_array_equal(grad, [[0, 1, 0], [0, -1, 0]])


def test_direct_momentum_balance():
    # Newton's third law: sum_i q_i grad(phi)_i = 0 (north_star invariant)
    pos, q = synth.generate("cube", 200, 7)
    phi, grad = oracle.direct(pos, q)
    tot = np.abs((q[:, None] * grad).sum(0)).max()
    assert tot <= 1e-12 * np.abs(q[:, None] * grad).sum()


def test_direct_shell_centre_exact():
    # every point of the sphere distribution is at radius 1 (up to rounding), so the
    # potential at the centre is sum q_j (shell at unit distance), up to rounding of r.
    pos, q = synth.generate("sphere", 500, 3)
    allp = np.vstack([pos, [[0.0, 0.0, 0.0]]])
    allq = np.concatenate([q, [0.0]])
    phi, grad = oracle.direct(allp, allq, targets=[500])
    assert abs(phi[0] - q.sum()) <= 1e-12 * np.abs(q).sum()
    # and the field at the centre is sum q_j x_j / |x_j|^3 = sum q_j x_j
    np.testing.assert_allclose(grad[0], (q[:, None] * pos).sum(0), rtol=0, atol=1e-12 * np.abs(q).sum())


def test_direct_shell_outside_monopole():
    # shell theorem: a uniform shell of total charge Q acts like Q at its centre outside.
    pos, _ = synth.generate("sphere", 20000, 5)
    q = np.full(len(pos), 1.0 / len(pos))
    x = np.array([[0.0, 0.0, 3.0]])
    phi, _ = oracle.direct(np.vstack([pos, x]), np.concatenate([q, [0.0]]), targets=[len(pos)])
    assert abs(phi[0] - 1.0 / 3.0) < 2e-3   # sampling noise of 20k random points


# ---------------------------------------------------------------- R2 - R4 --
def _spread_bits(v):
    # independent bit-interleave by magic-number spreading (not the oracle's per-level loop)
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def test_root_cube_and_keys_brute_force():
    pos, _ = synth.generate("plummer", 3000, 11)
    o, s, h = oracle.root_cube(pos)
    lo, hi = pos.min(0), pos.max(0)
    assert h == 0.5 * max(hi - lo)
    np.testing.assert_array_equal(o, (lo + hi) * 0.5 - h)
    assert s == 2.0 ** 20 / h
    # quantisation: floor((x - o) * s) clamped, computed here in numpy (same IEEE ops)
    i = np.clip(np.floor((pos - o) * s), 0, 2 ** 21 - 1).astype(np.uint64)
    ref = _spread_bits(i[:, 0]) | (_spread_bits(i[:, 1]) << np.uint64(1)) | (_spread_bits(i[:, 2]) << np.uint64(2))
    np.testing.assert_array_equal(oracle.keys(pos), ref)
    # every point quantises inside its cube cell: octant geometry check at level 3
    k = oracle.keys(pos)
    pref = (k >> np.uint64(3 * 18)).astype(np.int64)
    ix = sum(((pref >> (3 * l)) & 1) << l for l in range(3))
    iy = sum(((pref >> (3 * l + 1)) & 1) << l for l in range(3))
    iz = sum(((pref >> (3 * l + 2)) & 1) << l for l in range(3))
    w = 2 * h / 8
    for d, idx in enumerate([ix, iy, iz]):
        assert np.all(pos[:, d] >= o[d] + idx * w - 1e-12 * h)
        assert np.all(pos[:, d] <= o[d] + (idx + 1) * w + 1e-12 * h)


def test_key_spec_examples():
    # the minimum corner maps to key 0; a point in the (+x,+y,+z)
    # octant has level-1 digit 7.  Points chosen so the bounds are [0,1]^3.
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [0.9, 0.8, 0.7], [0.9, 0.1, 0.1], [0.1, 0.9, 0.1]])
    k = oracle.keys(pos)
    assert k[0] == 0
    assert k[1] == (1 << 63) - 1            # clamp to 2^21-1 on every axis
    assert (k[2] >> np.uint64(60)) == 7
    assert (k[3] >> np.uint64(60)) == 1     # +x only -> bit 0
    assert (k[4] >> np.uint64(60)) == 2     # +y only -> bit 1
    # prefix property: level-l digit path is the prefix of level l+1
    for kk in k:
        for l in range(1, 21):
            assert (int(kk) >> (3 * (21 - l))) == (int(kk) >> (3 * (21 - l - 1))) >> 3


# ------------------------------------------------------------------ R5 - R7 --
def _check_tree(f, pos, ncrit):
    c = f.cells()
    keys, perm = f.sorted()
    n = len(pos)
    # R5: stable sort, ties by original index
    k0 = oracle.keys(pos)
    order = np.lexsort((np.arange(n), k0))
    np.testing.assert_array_equal(perm, order)
    np.testing.assert_array_equal(keys, k0[order])
    # bijection
    assert sorted(perm.tolist()) == list(range(n))
    nc = len(c["level"])
    # R6: BFS (level, key) order, strictly ascending
    lk = list(zip(c["level"].tolist(), c["key"].tolist()))
    assert lk == sorted(lk) and len(set(lk)) == nc
    assert c["parent"][0] == -1 and c["body_begin"][0] == 0 and c["body_count"][0] == n
    sp = pos[perm]
    for i in range(nc):
        lvl, cnt, cb, cc = c["level"][i], c["body_count"][i], c["child_begin"][i], c["child_count"][i]
        assert (cc > 0) == (cnt > ncrit and lvl < 21)
        bb = c["body_begin"][i]
        # member particles share the cell key prefix
        assert np.all((keys[bb:bb + cnt] >> np.uint64(3 * (21 - lvl))) == c["key"][i])
        if cc:
            # children partition the parent's range, in digit order
            kids = range(cb, cb + cc)
            assert c["body_begin"][cb] == bb
            assert sum(c["body_count"][k] for k in kids) == cnt
            for k in kids:
                assert c["parent"][k] == i and c["level"][k] == lvl + 1
                assert (c["key"][k] >> np.uint64(3)) == c["key"][i]
                # tight box of a child inside the parent's
                assert np.all(c["bmin"][k] >= c["bmin"][i]) and np.all(c["bmax"][k] <= c["bmax"][i])
            for a, b in zip(kids, list(kids)[1:]):
                assert c["body_begin"][a] + c["body_count"][a] == c["body_begin"][b]
        # R7: tight box = exact min/max of members, centre, half-diagonal
        m = sp[bb:bb + cnt]
        np.testing.assert_array_equal(c["bmin"][i], m.min(0))
        np.testing.assert_array_equal(c["bmax"][i], m.max(0))
        np.testing.assert_array_equal(c["center"][i], (m.min(0) + m.max(0)) * 0.5)
        d = m.max(0) - m.min(0)
        assert c["radius"][i] == 0.5 * math.sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
    return c


@pytest.mark.parametrize("kind,n,ncrit", [("cube", 1000, 8), ("plummer", 2000, 16), ("sphere", 777, 5)])
def test_tree_invariants(kind, n, ncrit):
    pos, q = synth.generate(kind, n, 13)
    f = oracle.FMM(pos, q, 3, 0.5, ncrit)
    _check_tree(f, pos, ncrit)


def test_tree_octant_centres():
    # 8 bodies at the 8 octant centres, ncrit=1 -> root + 8 leaves
    pts = np.array([[x, y, z] for z in (0.25, 0.75) for y in (0.25, 0.75) for x in (0.25, 0.75)])
    f = oracle.FMM(pts, np.ones(8), 2, 0.5, 1)
    c = _check_tree(f, pts, 1)
    assert len(c["level"]) == 9 and c["child_count"][0] == 8
    assert np.all(c["child_count"][1:] == 0)
    np.testing.assert_array_equal(c["key"][1:], np.arange(8))


def test_tree_degenerate():
    # R20: N=1 -> single leaf, phi = 0; all-coincident -> chain to level 21
    f = oracle.FMM([[0.3, 0.2, 0.1]], [1.0], 4, 0.5, 1)
    assert f.counts()["ncell"] == 1
    phi, grad = f.evaluate()
    assert phi[0] == 0 and np.all(grad == 0)
    pts = np.full((5, 3), 0.25)
    f = oracle.FMM(pts, np.ones(5), 4, 0.5, 2)
    c = _check_tree(f, pts, 2)
    assert f.counts()["depth"] == 21 and len(c["level"]) == 22
    phi, grad = f.evaluate()
    assert np.all(phi == 0) and np.all(grad == 0)
    # N=0: no cells, no-op
    f = oracle.FMM(np.zeros((0, 3)), np.zeros(0), 4, 0.5, 2)
    assert f.counts()["ncell"] == 0
    phi, grad = f.evaluate()
    assert phi.shape == (0,)


def test_stable_sort_ties():
    # duplicated points: identical keys must keep original index order
    pos, q = synth.generate("cube", 100, 1)
    pos = np.vstack([pos, pos[::-1], pos[:10]])
    f = oracle.FMM(pos, np.ones(len(pos)), 2, 0.5, 4)
    _check_tree(f, pos, 4)


# ----------------------------------------------------------- R11 - R16 ------
def test_coefficient_order():
    e = oracle.multi_indices(3)
    assert e.tolist() == [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [2, 0, 0], [1, 1, 0], [1, 0, 1],
                          [0, 2, 0], [0, 1, 1], [0, 0, 2]]
    for P in (1, 4, 10, 16):
        assert oracle.ncoef(P) == P * (P + 1) * (P + 2) // 6 == len(oracle.multi_indices(P))


def test_p2m_closed_forms():
    # unit charge at the centre -> M_0 = 1, all others 0
    M = oracle.p2m(6, [[0.1, 0.2, 0.3]], [1.0], [0.1, 0.2, 0.3])
    assert M[0] == 1.0 and np.all(M[1:] == 0)
    # +1 at c+a, -1 at c-a: odd moments 2 a^b/b!, even moments 0
    a = np.array([0.1, -0.05, 0.02])
    M = oracle.p2m(5, [a, -a], [1.0, -1.0], [0, 0, 0])
    ex = oracle.multi_indices(5)
    for k, e in enumerate(ex):
        expect = 0.0 if e.sum() % 2 == 0 else 2 * np.prod(a ** e) / np.prod([math.factorial(v) for v in e])
        assert abs(M[k] - expect) <= 1e-16


def test_m2m_exact():
    # M2M is exact in the Cartesian basis: M2M(P2M at child centre) == P2M at parent centre
    rng = np.random.default_rng(1)
    pts = rng.random((30, 3)) * 0.1
    q = rng.uniform(-1, 1, 30)
    cc, cp = np.array([0.05, 0.04, 0.06]), np.array([0.1, 0.12, 0.08])
    for P in (1, 4, 10):
        Mc = oracle.p2m(P, pts, q, cc)
        Mp = oracle.m2m(P, Mc, cc - cp)
        ref = oracle.p2m(P, pts, q, cp)
        assert np.abs(Mp - ref).max() <= 1e-13 * np.abs(ref).max()
    # shift 0 is the identity; pure monopole shifted by d -> q d^a/a!
    M = oracle.m2m(4, Mc[:20], [0, 0, 0])
    np.testing.assert_array_equal(M, Mc[:20])


def test_deriv_closed_forms(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "closed_forms.json")))["deriv_at_123"]
    D = oracle.deriv(5, g["d"])
    ex = oracle.multi_indices(5).tolist()
    for ent in g["entries"]:
        k = ex.index(ent["gamma"])
        ref = eval(ent["value_expr"], {"sqrt": math.sqrt})
        assert abs(D[k] - ref) <= 1e-15 * abs(ref) + 1e-18, ent


def test_deriv_harmonic_and_finite_difference():
    # Laplace: sum_i D^{gamma + 2e_i} G = 0 for every gamma (exact, any order)
    P = 12
    d = np.array([0.7, -0.4, 1.1])
    D = oracle.deriv(P, d)
    ex = oracle.multi_indices(P).tolist()
    idx = {tuple(e): k for k, e in enumerate(ex)}
    for e in ex:
        if sum(e) > P - 3:
            continue
        s = sum(D[idx[tuple(np.add(e, 2 * np.eye(3, dtype=int)[i]))]] for i in range(3))
        big = max(abs(D[idx[tuple(np.add(e, 2 * np.eye(3, dtype=int)[i]))]]) for i in range(3))
        assert abs(s) <= 1e-13 * big
    # finite differences: d/dx_i D^gamma = D^{gamma+e_i} (central, step 1e-5)
    hstep = 1e-5
    for i in range(3):
        dp, dm = d.copy(), d.copy()
        dp[i] += hstep; dm[i] -= hstep
        fd = (oracle.deriv(P, dp) - oracle.deriv(P, dm)) / (2 * hstep)
        for e in ex:
            if sum(e) > P - 2:
                continue
            k1 = idx[tuple(np.add(e, np.eye(3, dtype=int)[i]))]
            assert abs(fd[idx[tuple(e)]] - D[k1]) <= 1e-6 * max(1.0, abs(D[k1]))


def test_m2l_monopole(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "closed_forms.json")))["m2l_monopole"]
    P = 4
    M = np.zeros(oracle.ncoef(P)); M[0] = g["q"]
    L = oracle.m2l(P, M, [-g["d"], 0, 0])          # d = c_A - c_B, source at +x
    ex = oracle.multi_indices(P).tolist()
    assert abs(L[0] - g["L0"]) < 1e-15
    assert abs(L[ex.index([1, 0, 0])] - g["Lx"]) < 1e-15
    assert abs(L[ex.index([2, 0, 0])] - g["Lxx"]) < 1e-15
    assert abs(L[ex.index([0, 2, 0])] - g["Lyy"]) < 1e-15


def test_m2l_chain_decays_with_P():
    # P2M -> M2L -> L2P against the direct far field decreases with P (PAPER.md:187 O(theta^P))
    rng = np.random.default_rng(3)
    src = rng.random((20, 3)) * 0.2
    q = rng.uniform(-1, 1, 20)
    tgt = rng.random((10, 3)) * 0.2 + np.array([1.0, 0.2, 0.1])
    cs, ct = np.full(3, 0.1), np.array([1.1, 0.3, 0.2])
    phid, gradd = oracle.p2p(tgt, src, q)
    errs, gerrs = [], []
    for P in (2, 4, 6, 8, 10):
        M = oracle.p2m(P, src, q, cs)
        L = oracle.m2l(P, M, ct - cs)
        phi, grad = oracle.l2p(P, L, ct, tgt)
        errs.append(oracle.rel_l2(phi, phid)); gerrs.append(oracle.rel_l2(grad, gradd))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert all(b < a for a, b in zip(gerrs, gerrs[1:])), gerrs
    assert errs[-1] < 1e-7


def test_l2l_then_l2p_equals_l2p():
    # L2L is an exact re-centring of the local polynomial
    rng = np.random.default_rng(4)
    for P in (1, 3, 8):
        L = rng.normal(size=oracle.ncoef(P))
        cp, cc = np.array([0.5, 0.5, 0.5]), np.array([0.6, 0.45, 0.52])
        pts = cc + rng.uniform(-0.05, 0.05, (7, 3))
        phi_p, g_p = oracle.l2p(P, L, cp, pts)
        Lc = oracle.l2l(P, L, cc - cp)
        phi_c, g_c = oracle.l2p(P, Lc, cc, pts)
        assert oracle.rel_l2(phi_c, phi_p) < 1e-13 and oracle.rel_l2(g_c, g_p) < 1e-13 or P == 1


def test_l2p_closed_forms_and_gradient():
    P = 6
    L = np.zeros(oracle.ncoef(P))
    phi, grad = oracle.l2p(P, L, [0, 0, 0], [[0.1, 0.2, 0.3]])
    assert phi[0] == 0 and np.all(grad == 0)
    L[0] = 2.5
    phi, grad = oracle.l2p(P, L, [0, 0, 0], [[0.1, 0.2, 0.3], [1, 2, 3]])
    np.testing.assert_array_equal(phi, [2.5, 2.5]); assert np.all(grad == 0)
    # the gradient is the exact derivative of the degree-(P-1) local polynomial
    rng = np.random.default_rng(5)
    L = rng.normal(size=oracle.ncoef(P))
    x = np.array([[0.03, -0.02, 0.05]])
    _, g = oracle.l2p(P, L, [0, 0, 0], x)
    for i in range(3):
        e = np.zeros((1, 3)); e[0, i] = 1e-6
        fd = (oracle.l2p(P, L, [0, 0, 0], x + e)[0] - oracle.l2p(P, L, [0, 0, 0], x - e)[0]) / 2e-6
        assert abs(fd[0] - g[0, i]) < 1e-8
    # P = 1: far-field gradient is 0
    _, g = oracle.l2p(1, [3.0], [0, 0, 0], x)
    assert np.all(g == 0)


# ------------------------------------------------------------------ R8 - R10 -
def test_mac_spec_examples():
    # SPEC.md:286-288, via two single-body cells: R = 0 cells at any distance -> M2L
    f = oracle.FMM([[0, 0, 0], [1, 0, 0]], [1.0, 1.0], 2, 0.4, 1).traverse()
    m2l, p2p = f.lists()
    assert f.counts()["ncell"] == 3
    assert m2l.tolist() == [[1, 2], [2, 1]] and p2p.tolist() == [[1, 1], [2, 2]]   # self pairs: d = 0
    # one overlapping leaf -> exactly one P2P (self pair)
    f = oracle.FMM([[0, 0, 0], [1, 0, 0]], [1.0, 1.0], 2, 0.4, 5).traverse()
    m2l, p2p = f.lists()
    assert len(m2l) == 0 and p2p.tolist() == [[0, 0]]


def _coverage(f, n):
    """count, for every (target i, source j) body pair, how many list entries cover it"""
    c = f.cells()
    _, perm = f.sorted()
    m2l, p2p = f.lists()
    cov = np.zeros((n, n), dtype=np.int32)
    for a, b in np.vstack([m2l, p2p]):
        ia = slice(c["body_begin"][a], c["body_begin"][a] + c["body_count"][a])
        ib = slice(c["body_begin"][b], c["body_begin"][b] + c["body_count"][b])
        cov[ia, ib] += 1
    return cov, c, m2l, p2p


@pytest.mark.parametrize("kind,n,ncrit,theta", [("cube", 512, 8, 0.4), ("plummer", 700, 4, 0.6),
                                                ("sphere", 300, 3, 0.3)])
def test_dtt_exactly_once_and_mac(kind, n, ncrit, theta):
    pos, q = synth.generate(kind, n, 21)
    f = oracle.FMM(pos, q, 3, theta, ncrit).traverse()
    cov, c, m2l, p2p = _coverage(f, n)
    assert np.all(cov == 1)          # every body pair covered exactly once
    for a, b in m2l:                 # every M2L satisfies the MAC strictly
        d = np.linalg.norm(c["center"][a] - c["center"][b])
        assert c["radius"][a] + c["radius"][b] < theta * d
    for a, b in p2p:
        assert c["child_count"][a] == 0 and c["child_count"][b] == 0
    # canonical order, no duplicates (R10)
    for lst in (m2l, p2p):
        t = [tuple(x) for x in lst.tolist()]
        assert t == sorted(set(t))


def test_dtt_bfs_frontier_same_set():
    # R9 is a pure function of the pair: a breadth-first traversal emits the same sets
    pos, q = synth.generate("plummer", 1500, 8)
    theta = 0.45
    f = oracle.FMM(pos, q, 3, theta, 10).traverse()
    c = f.cells()
    m2l, p2p = f.lists()
    leaf = c["child_count"] == 0
    fr = [(0, 0)]
    bm, bp = [], []
    while fr:
        nxt = []
        for a, b in fr:
            dx = c["center"][a] - c["center"][b]
            if c["radius"][a] + c["radius"][b] < theta * math.sqrt((dx[0] * dx[0] + dx[1] * dx[1]) + dx[2] * dx[2]):
                bm.append((a, b))
            elif leaf[a] and leaf[b]:
                bp.append((a, b))
            elif leaf[b] or (not leaf[a] and c["radius"][a] >= c["radius"][b]):
                nxt += [(k, b) for k in range(c["child_begin"][a], c["child_begin"][a] + c["child_count"][a])]
            else:
                nxt += [(a, k) for k in range(c["child_begin"][b], c["child_begin"][b] + c["child_count"][b])]
        fr = nxt
    assert sorted(bm) == [tuple(x) for x in m2l.tolist()]
    assert sorted(bp) == [tuple(x) for x in p2p.tolist()]


# ------------------------------------------------------------- end to end ---
def test_single_leaf_equals_direct():
    # ncrit >= N: one leaf, one self P2P -> identical to the direct sum
    pos, q = synth.generate("cube", 300, 2)
    f = oracle.FMM(pos, q, 4, 0.5, 300)
    phi, grad = f.evaluate()
    dp, dg = oracle.direct(pos, q)
    assert oracle.rel_l2(phi, dp) <= 1e-14 and oracle.rel_l2(grad, dg) <= 1e-14


def test_tiny_theta_equals_direct():
    # theta -> 0: MAC never accepts, P2P only -> direct sum
    pos, q = synth.generate("plummer", 400, 4)
    f = oracle.FMM(pos, q, 4, 1e-3, 8).traverse()
    c = f.cells()
    m2l, _ = f.lists()
    # the only accepted pairs are point cells (R = 0), for which M2L is exact
    assert np.all(c["radius"][m2l[:, 0]] == 0) and np.all(c["radius"][m2l[:, 1]] == 0)
    phi, grad = f.evaluate()
    dp, dg = oracle.direct(pos, q)
    assert oracle.rel_l2(phi, dp) <= 1e-14 and oracle.rel_l2(grad, dg) <= 1e-14


def test_n2_exact():
    f = oracle.FMM([[0.1, 0.2, 0.3], [0.4, 0.1, -0.2]], [1.0, -2.0], 4, 0.5, 1)
    phi, grad = f.evaluate()
    dp, dg = oracle.direct([[0.1, 0.2, 0.3], [0.4, 0.1, -0.2]], [1.0, -2.0])
    assert oracle.rel_l2(phi, dp) <= 1e-14 and oracle.rel_l2(grad, dg) <= 1e-14


def test_error_decreases_with_P():
    # error vs direct sum strictly decreases over P in {4,6,8,10} at theta=0.4,
    # with err(10)/err(4) <= 1e-2; plus the momentum invariant (north_star)
    n = 6000
    pos, q = synth.generate("cube", n, 9)
    t = synth.sample_targets(n, 400, 9)
    dp, dg = oracle.direct(pos, q, t)
    errs = []
    for P in (4, 6, 8, 10):
        f = oracle.FMM(pos, q, P, 0.4, 64)
        phi, grad = f.evaluate(t)
        errs.append(oracle.rel_l2(phi, dp))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] / errs[0] <= 1e-2, errs


def test_momentum_fmm():
    n = 3000
    pos, q = synth.generate("cube", n, 12)
    f = oracle.FMM(pos, q, 6, 0.5, 32)
    phi, grad = f.evaluate()
    dp, dg = oracle.direct(pos, q)
    err = oracle.rel_l2(grad, dg)
    mom = np.abs((q[:, None] * grad).sum(0)).max() / np.abs(q[:, None] * grad).sum()
    assert mom <= 10 * err


def test_single_far_source_bound():
    # a cluster of targets and one far source: phi_i = q/|x_i - y| within (rho_t/D)^P (north_star)
    rng = np.random.default_rng(9)
    tg = rng.uniform(-0.05, 0.05, (64, 3))
    y = np.array([3.0, 1.0, -2.0])
    pos = np.vstack([tg, y]); q = np.concatenate([np.zeros(64), [0.7]])
    D = np.linalg.norm(y)
    for P in (3, 6, 9):
        f = oracle.FMM(pos, q, P, 0.3, 64 if False else 63)
        phi, _ = f.evaluate(np.arange(64))
        exact = 0.7 / np.linalg.norm(tg - y, axis=1)
        rho = np.linalg.norm(tg - tg.mean(0), axis=1).max() * 2
        assert np.abs(phi - exact).max() <= 0.7 / (D - rho) * (rho / (D - rho)) ** P * 10


def test_sampled_mode_bitwise_equals_full():
    pos, q = synth.generate("plummer", 3000, 6)
    f = oracle.FMM(pos, q, 5, 0.5, 16)
    phi, grad = f.evaluate()
    t = synth.sample_targets(3000, 50, 6)
    phs, grs = oracle.FMM(pos, q, 5, 0.5, 16).evaluate(t)
    np.testing.assert_array_equal(phs, phi[t])
    np.testing.assert_array_equal(grs, grad[t])


def test_bad_arguments():
    pos, q = synth.generate("cube", 10, 1)
    for P, th, nc in [(0, 0.5, 4), (17, 0.5, 4), (4, 0.0, 4), (4, 1.0, 4), (4, 0.5, 0)]:
        with pytest.raises(ValueError):
            oracle.FMM(pos, q, P, th, nc)


def test_generator_determinism_and_plummer_median():
    a = synth.generate("plummer", 20000, 5)
    b = synth.generate("plummer", 20000, 5)
    np.testing.assert_array_equal(a[0], b[0])
    r = np.linalg.norm(a[0], axis=1)
    # truncated Plummer (a=1, r<=100): median radius where m(r)/m(100) = 1/2
    mmax = 100 ** 3 / (100 ** 2 + 1) ** 1.5
    rh = 1 / math.sqrt((0.5 * mmax) ** (-2 / 3) - 1)
    assert abs(np.median(r) / rh - 1) < 0.03 and r.max() <= 100
    s = synth.generate("sphere", 100, 1)[0]
    assert np.all(np.abs(np.linalg.norm(s, axis=1) - 1) < 1e-12)
    c = synth.generate("cube", 100, 1)
    assert np.all((c[0] >= 0) & (c[0] < 1)) and np.all((c[1] >= -1) & (c[1] < 1))
    f32 = synth.generate("cube", 100, 1, np.float32)[0]
    np.testing.assert_array_equal(f32, c[0].astype(np.float32))


# ------------------------------------------------------ per-partition mode (§8e) --
def _partitions(pos, k):
    return np.array_split(np.argsort(pos[:, 0], kind="stable"), k)


def _global_bounds(pos):
    return np.concatenate([pos.min(0), pos.max(0)])


@pytest.mark.parametrize("glob", [False, True])
def test_partition_tiny_theta_equals_direct(glob):
    # theta -> 0: every cross-partition pair is P2P, so the multi-tree sum is the direct sum
    pos, q = synth.generate("plummer", 900, 31)
    parts = _partitions(pos, 3)
    b = _global_bounds(pos) if glob else None
    trees = [oracle.FMM(pos[p], q[p], 3, 1e-3, 8, bounds=b) for p in parts]
    dp, dg = oracle.direct(pos, q)
    for k, p in enumerate(parts):
        phi, g = oracle.evaluate_multi(trees[k], [t for j, t in enumerate(trees) if j != k])
        assert oracle.rel_l2(phi, dp[p]) <= 1e-13 and oracle.rel_l2(g, dg[p]) <= 1e-13


@pytest.mark.parametrize("glob", [False, True])
def test_partition_exactly_once_coverage(glob):
    # local lists of tree k plus its remote lists against every other tree cover each
    # (target body, source body) pair of the whole system exactly once
    pos, q = synth.generate("cube", 600, 32)
    parts = _partitions(pos, 3)
    b = _global_bounds(pos) if glob else None
    trees = [oracle.FMM(pos[p], q[p], 3, 0.5, 8, bounds=b).traverse() for p in parts]
    for k in range(3):
        T = trees[k]
        cT = T.cells()
        _, permT = T.sorted()
        cov = np.zeros((len(parts[k]), len(pos)), dtype=np.int32)
        for j in range(3):
            S = trees[j]
            cS = S.cells()
            _, permS = S.sorted()
            m2l, p2p = T.lists() if j == k else oracle.traverse_pair(T, S)
            for a, b in np.vstack([m2l, p2p]):
                ta = permT[cT["body_begin"][a]:cT["body_begin"][a] + cT["body_count"][a]]
                sb = parts[j][permS[cS["body_begin"][b]:cS["body_begin"][b] + cS["body_count"][b]]]
                cov[np.ix_(ta, sb)] += 1
            if j != k:
                for a, b in m2l:   # remote M2L pairs satisfy the MAC strictly
                    d = np.linalg.norm(cT["center"][a] - cS["center"][b])
                    assert cT["radius"][a] + cS["radius"][b] < 0.5 * d
        assert np.all(cov == 1)


def test_partition_single_tree_equals_evaluate():
    pos, q = synth.generate("cube", 800, 33)
    a = oracle.FMM(pos, q, 5, 0.5, 16)
    b = oracle.FMM(pos, q, 5, 0.5, 16)
    phi1, g1 = a.evaluate()
    phi2, g2 = oracle.evaluate_multi(b, [])
    np.testing.assert_array_equal(phi1, phi2)
    np.testing.assert_array_equal(g1, g2)


def test_root_bounds_own_box_is_default():
    pos, q = synth.generate("plummer", 700, 34)
    a = oracle.FMM(pos, q, 4, 0.5, 16)
    b = oracle.FMM(pos, q, 4, 0.5, 16, bounds=_global_bounds(pos))
    for x, y in zip(a.sorted(), b.sorted()):
        np.testing.assert_array_equal(x, y)
    for k, v in a.cells().items():
        np.testing.assert_array_equal(v, b.cells()[k])
    np.testing.assert_array_equal(a.evaluate()[0], b.evaluate()[0])


def test_root_bounds_global_keys_are_subtree_keys():
    # HOT reading (DESIGN.md §2 reading 9): a Morton-range part built on the global root cube
    # has exactly the global keys, and every one of its cells is a cell of the global octree
    pos, q = synth.generate("cube", 3000, 35)
    gk = oracle.keys(pos)
    b = _global_bounds(pos)
    order = np.argsort(gk, kind="stable")
    part = np.sort(order[1000:2000])              # one Morton range of the global curve
    t = oracle.FMM(pos[part], q[part], 4, 0.5, 16, bounds=b)
    k, perm = t.sorted()
    np.testing.assert_array_equal(k, gk[part][perm])
    c = t.cells()
    lo = c["body_begin"]; lv = c["level"]
    for i in range(len(lv)):                     # cell key = common level-l prefix of its bodies
        pre = k[lo[i]] >> np.uint64(3 * (21 - lv[i]))
        assert c["key"][i] == pre


def test_root_bounds_reject_outside():
    pos, q = synth.generate("cube", 10, 36)
    with pytest.raises(ValueError):
        oracle.FMM(pos, q, 3, 0.5, 4, bounds=np.array([0.1, 0.1, 0.1, 0.9, 0.9, 0.9]))
