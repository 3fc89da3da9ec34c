"""Host-side logic of the multi-GPU driver on CPU (no GPU): the library's partition rules
(fmm_splitters, fmm_orb_plan, fmm_alpha_tuner_*; csrc/dist.cu) driven through their callback
entry points, and the same rules over a world_size-2 gloo process group: each process holds half
of the particles, its histogram callback all-reduces over gloo -- the N>1 partition step the
driver runs over NCCL -- and both ranks must agree on the splitters and the ORB boxes.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_1405_7487_b200.dist import partition_splitters


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _host_hist_fn(keys, w=None):
    """numpy stand-in for the all-reduced device histogram (same binning as fmm_part_histogram)."""
    w = np.ones(len(keys)) if w is None else w

    def fn(prefixes, pbits, bits):
        out = np.zeros((len(prefixes), 1 << bits))
        lo = np.uint64(63 - pbits - bits)
        for r, pre in enumerate(prefixes):
            sel = np.ones(len(keys), bool) if pbits == 0 else (keys >> np.uint64(63 - pbits)) == np.uint64(pre)
            b = ((keys[sel] >> lo) & np.uint64((1 << bits) - 1)).astype(np.int64)
            out[r] = np.bincount(b, weights=w[sel], minlength=1 << bits)
        return out
    return fn


@pytest.mark.parametrize("kind", ["cube", "plummer"])
def test_partition_gives_balanced_morton_ranges(kind):
    # Plummer: the top 16 key bits put most particles in a few bins; refinement splits them
    pos, _ = synth.generate(kind, 20000, 5)
    k = oracle.keys(pos)
    order = np.argsort(k, kind="stable")
    for K in (1, 2, 3, 4, 8):
        spl = partition_splitters(_host_hist_fn(k), K)
        assert len(spl) == K - 1 and np.all(np.diff(spl.astype(np.float64)) >= 0)
        dest = np.searchsorted(spl, k, side="right")     # = number of splitters <= key
        assert np.all(np.diff(dest[order]) >= 0)           # contiguous along the Morton curve
        cnt = np.bincount(dest, minlength=K)
        assert np.abs(cnt - len(pos) / K).max() <= 0.01 * len(pos) / K + 1, cnt


def test_partition_weighted():
    # Eq. (1): weights move the cuts -- heavy particles get ranks of their own
    pos, _ = synth.generate("cube", 4000, 6)
    k = oracle.keys(pos)
    w = np.where(pos[:, 0] < 0.25, 9.0, 1.0)
    spl = partition_splitters(_host_hist_fn(k, w), 4)
    dest = np.searchsorted(spl, k, side="right")
    share = np.array([w[dest == j].sum() for j in range(4)]) / w.sum()
    assert np.abs(share - 0.25).max() < 0.01, share


def test_partition_degenerate():
    k = np.full(100, np.uint64(12345), dtype=np.uint64)   # coincident particles: one key
    spl = partition_splitters(_host_hist_fn(k), 4)
    dest = np.searchsorted(spl, k, side="right")
    assert len(np.unique(dest)) == 1                        # equal keys never split


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_1405_7487_b200.dist import orb_plan
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pos, _ = synth.generate("plummer", 20000, 5)
        mine = slice(rank * 10000, (rank + 1) * 10000)           # this process's particles
        k = oracle.keys(pos)[mine]
        local = _host_hist_fn(k)

        def global_hist(prefixes, pbits, bits):               # the all-reduce the driver does
            h = torch.from_numpy(np.ascontiguousarray(local(prefixes, pbits, bits)))
            dist.all_reduce(h)
            return h.numpy()
        spl = partition_splitters(global_hist, 4)
        xyz = _coords(k)
        grp = np.zeros(len(k), dtype=np.int64)

        def orb_hist(axis, prefix, pbits, bits):
            out = np.zeros((4, 1 << bits))
            for g in range(4):
                if axis[g] < 0:
                    continue
                c = xyz[:, axis[g]]
                sel = grp == g
                if pbits:
                    sel &= (c >> (21 - pbits)) == prefix[g]
                out[g] = np.bincount((c[sel] >> (21 - pbits - bits)) & ((1 << bits) - 1), minlength=1 << bits)
            h = torch.from_numpy(out)
            dist.all_reduce(h)
            return h.numpy()

        def orb_split(axis, cut, right):
            for g in range(4):
                if axis[g] >= 0:
                    grp[(grp == g) & (xyz[:, axis[g]] >= cut[g])] = right[g]
        boxes = orb_plan(orb_hist, orb_split, 4)
        q.put((rank, spl.tolist(), {r: (b["lo"], b["hi"]) for r, b in boxes.items()},
               np.bincount(np.searchsorted(spl, k, side="right"), minlength=4).tolist(),
               np.bincount(grp, minlength=4).tolist()))
    finally:
        dist.destroy_process_group()


def test_partition_rules_over_gloo():
    """world_size 2 (gloo): the driver's splitter and ORB rules with globally all-reduced
    histograms give both ranks the same splitters and boxes, equal to the single-process rules
    on all particles, and balanced global shares."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=180)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    pos, _ = synth.generate("plummer", 20000, 5)
    k = oracle.keys(pos)
    assert res[0][1] == partition_splitters(_host_hist_fn(k), 4).tolist()
    cnt = np.array(res[0][3]) + np.array(res[1][3])
    assert np.abs(cnt - 5000).max() <= 0.01 * 5000 + 1, cnt
    ocnt = np.array(res[0][4]) + np.array(res[1][4])
    assert np.abs(ocnt - 5000).max() <= 0.01 * 5000 + 1, ocnt


def _coords(keys):
    """R3 quantised coordinates from 63-bit Morton keys (x -> bit 0 of each octal digit)."""
    out = np.zeros((len(keys), 3), dtype=np.int64)
    for a in range(3):
        c = np.zeros(len(keys), dtype=np.int64)
        for l in range(21):
            c |= (((keys >> np.uint64(3 * l + a)) & np.uint64(1)).astype(np.int64)) << l
        out[:, a] = c
    return out


@pytest.mark.parametrize("K", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("kind", ["cube", "plummer"])
def test_orb_plan_balanced_boxes(K, kind):
    from paper_1405_7487_b200.dist import orb_plan
    pos, _ = synth.generate(kind, 12000, 9)
    xyz = _coords(oracle.keys(pos))
    w = 1.0 + (pos[:, 0] > np.median(pos[:, 0]))          # uneven weights
    grp = np.zeros(len(pos), dtype=np.int64)

    def hist_fn(axis, prefix, pbits, bits):
        out = np.zeros((K, 1 << bits))
        for g in range(K):
            if axis[g] < 0:
                continue
            c = xyz[:, axis[g]]
            sel = grp == g
            if pbits:
                sel &= (c >> (21 - pbits)) == prefix[g]
            b = (c[sel] >> (21 - pbits - bits)) & ((1 << bits) - 1)
            out[g] = np.bincount(b, weights=w[sel], minlength=1 << bits)
        return out

    def split_fn(axis, cut, right):
        for g in range(K):
            if axis[g] >= 0:
                m = (grp == g) & (xyz[:, axis[g]] >= cut[g])
                grp[m] = right[g]

    groups = orb_plan(hist_fn, split_fn, K)
    assert sorted(groups) == list(range(K))
    share = np.array([w[grp == r].sum() for r in range(K)]) / w.sum()
    assert np.abs(share - 1.0 / K).max() < 0.01, share
    for r, g in groups.items():               # every particle lies in its rank's box
        m = grp == r
        assert np.all((xyz[m] >= np.array(g["lo"])) & (xyz[m] < np.array(g["hi"])))


def _run_tuner(cost, steps, **kw):
    """Drive the library's alpha tuner the way fmm_dist_solve does: alpha_k is set before step k's
    weights, and step k's runtime reflects the partition made with alpha_{k-1}."""
    from paper_1405_7487_b200.dist import AlphaTuner
    tu = AlphaTuner(**kw)
    prev = None
    for _ in range(steps):
        a = tu.next_alpha()
        tu.report(cost(prev if prev is not None else 1.0))
        prev = a
    return tu


@pytest.mark.parametrize("amin", [0.08, 0.3, 1.0, 6.0])
def test_alpha_tuner_finds_minimum(amin):
    """Golden-section over log(alpha) ("optimized over the time steps to minimize the
    total runtime"): on a unimodal runtime with its minimum at amin it converges to amin, scoring
    each probe by the step after the one that set it."""
    cost = lambda a: 1.0 + (np.log(a) - np.log(amin)) ** 2
    tu = _run_tuner(cost, 80, lo=1.0 / 16, hi=16.0, tol=0.05)
    assert tu.converged
    assert abs(np.log(tu.best) - np.log(amin)) < 0.1, (tu.best, amin, tu.history)
    # every scored probe's runtime is the cost of the alpha it was scored for (no lag mix-up)
    for a, t in tu.history:
        assert t == pytest.approx(cost(a))
    # golden-section: ~log(range/tol)/log(1/0.618) probes, two steps each
    assert len(tu.history) <= 16


def test_alpha_tuner_edges():
    from paper_1405_7487_b200.dist import AlphaTuner
    with pytest.raises(ValueError):
        AlphaTuner(lo=2.0, hi=1.0)
    with pytest.raises(ValueError):
        AlphaTuner(lo=0.0, hi=1.0)
    # monotone runtime: converges to the bracket end
    tu = _run_tuner(lambda a: a, 80, lo=0.1, hi=10.0, tol=0.05)
    assert tu.converged and tu.best < 0.13
    tu = _run_tuner(lambda a: -a, 80, lo=0.1, hi=10.0, tol=0.05)
    assert tu.converged and tu.best > 7.5
    # after convergence alpha is frozen at the best probe
    a = tu.next_alpha()
    tu.report(123.0)
    assert tu.next_alpha() == a
