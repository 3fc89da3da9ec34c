"""Multi-GPU FMM: Morton-range partition + local essential tree (LET) exchange.

One process per GPU.  Every step on the particle and tree data runs in libfmm's kernels
(part.cu, let.cu and the single-GPU path); this module only sequences the calls and moves
the byte messages between ranks through a `Comm`:

* `TorchComm`     -- torch.distributed (NCCL on B200s: all_to_all_single with uneven splits is
                     NCCL grouped send/recv; gloo for the CPU plumbing tests);
* `LoopbackComm`  -- K ranks driven by ONE process on one device (single-GPU parity tests):
                     the ranks run one after another, messages are handed over in memory.
                     Nothing waits on another rank's kernels, so this is safe on one GPU.

Collectives take and return one entry per rank this process drives.

The step (§II-B/C):
  1. global bounds = all-reduce of fmm_bounds; keys under the global root cube (R2-R4);
  2. weighted key histogram (Eq. (1) weights; 1 at the first step),
     all-reduced; rank j takes the bins whose cumulative weight falls in [j/K, (j+1)/K);
  3. particles exchanged to their ranks (fmm_part_pack + all-to-all);
  4. local tree from the LOCAL bounds; covers all-gathered; each rank packs
     for every peer the part of its tree that peer can need (fmm_let_plan/pack_struct);
  5. LET structure sent in K-1 ring rounds of grouped send/recv: the local dual tree traversal
     overlaps round 1 and every received fragment is grafted and traversed from (local root,
     remote root) while the next round is in flight; then the
     canonical lists;
  6. upward pass, multipole/charge all-to-all, unpack, M2L + P2P + downward;
  7. results returned to the particles' owners in their original order.
"""
from __future__ import annotations

import time

import numpy as np
import torch

from .costs import m2l_cost_ratio
from .fmm import FMM

HIST_BITS = 16


# ------------------------------------------------------------------ communication
class Comm:
    world: int
    ranks: list   # global ranks driven by this process

    def allreduce(self, xs, op):   # op in {"sum", "min", "max"}
        raise NotImplementedError

    def allgather(self, xs):       # -> per local rank, list over all ranks
        raise NotImplementedError

    def alltoallv(self, sends, async_op=False):
        """sends[i][j]: 1-D tensor from local rank i to global rank j.  Returns recv with
        recv[i][j] from global rank j (or a handle whose wait() returns it)."""
        raise NotImplementedError

    def sendrecv(self, sends, dst, src, recv_sizes, async_op=False):
        """Point-to-point round: local rank i sends sends[i] to global rank dst[i] and receives
        recv_sizes[i] elements from global rank src[i] (grouped send/recv, deadlock-free)."""
        raise NotImplementedError

    def barrier(self):
        pass


class _Done:
    def __init__(self, v):
        self.v = v

    def wait(self):
        return self.v


class LoopbackComm(Comm):
    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def allreduce(self, xs, op):
        st = torch.stack(xs)
        r = {"sum": st.sum(0), "min": st.min(0).values, "max": st.max(0).values}[op]
        return [r.clone() for _ in xs]

    def allgather(self, xs):
        return [list(xs) for _ in xs]

    def alltoallv(self, sends, async_op=False):
        recv = [[sends[j][i] for j in range(self.world)] for i in range(self.world)]
        return _Done(recv) if async_op else recv

    def sendrecv(self, sends, dst, src, recv_sizes, async_op=False):
        by_dst = {dst[j]: j for j in range(self.world)}
        recv = [sends[by_dst[i]] for i in range(self.world)]
        assert all(src[i] == by_dst[i] and recv[i].numel() == recv_sizes[i] for i in range(self.world))
        return _Done(recv) if async_op else recv


class _P2PWork:
    def __init__(self, works, out):
        self.works, self.out = works, out

    def wait(self):
        for w in self.works:
            w.wait()
        return [self.out]


class _A2AWork:
    def __init__(self, work, out, sizes):
        self.work, self.out, self.sizes = work, out, sizes

    def wait(self):
        if self.work is not None:
            self.work.wait()
        return [list(self.out.split(self.sizes))]


class TorchComm(Comm):
    """One rank per process over an initialised torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def allreduce(self, xs, op):
        d = self.dist
        t = xs[0].clone()
        d.all_reduce(t, op={"sum": d.ReduceOp.SUM, "min": d.ReduceOp.MIN, "max": d.ReduceOp.MAX}[op], group=self.group)
        return [t]

    def allgather(self, xs):
        out = [torch.empty_like(xs[0]) for _ in range(self.world)]
        self.dist.all_gather(out, xs[0].contiguous(), group=self.group)
        return [out]

    def alltoallv(self, sends, async_op=False):
        s = sends[0]
        dev = s[0].device
        in_sizes = [int(t.numel()) for t in s]
        out_sz = torch.empty(self.world, dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(out_sz, torch.tensor(in_sizes, dtype=torch.int64, device=dev), group=self.group)
        sizes = [int(v) for v in out_sz.tolist()]
        inp = torch.cat([t.reshape(-1) for t in s])
        out = torch.empty(sum(sizes), dtype=s[0].dtype, device=dev)
        work = self.dist.all_to_all_single(out, inp, output_split_sizes=sizes, input_split_sizes=in_sizes,
                                           group=self.group, async_op=async_op)
        h = _A2AWork(work if async_op else None, out, sizes)
        return h if async_op else h.wait()

    def sendrecv(self, sends, dst, src, recv_sizes, async_op=False):
        d = self.dist
        t = sends[0]
        out = torch.empty(int(recv_sizes[0]), dtype=t.dtype, device=t.device)
        ops = []
        if t.numel():
            ops.append(d.P2POp(d.isend, t, dst[0], group=self.group))
        if out.numel():
            ops.append(d.P2POp(d.irecv, out, src[0], group=self.group))
        works = d.batch_isend_irecv(ops) if ops else []
        h = _P2PWork(works, out)
        return h if async_op else h.wait()

    def barrier(self):
        self.dist.barrier(group=self.group)


# ------------------------------------------------------------------ host logic
def choose_bins(hist: np.ndarray, targets: np.ndarray):
    """For each target weight t (measured from the start of this histogram): the bin where
    the inclusive cumulative weight first reaches t, and the weight still needed inside it."""
    c = np.cumsum(np.asarray(hist, dtype=np.float64))
    b = np.minimum(np.searchsorted(c, targets, side="left"), len(c) - 1)
    before = np.where(b > 0, c[np.maximum(b - 1, 0)], 0.0)
    return b.astype(np.int64), np.asarray(targets, dtype=np.float64) - before


def partition_splitters(hist_fn, nranks: int, bits: int = HIST_BITS, tol: float = 1.0 / 512):
    """Morton-range splitters by histogram refinement ("HOT is analogous to radix
    sort, where each bit of the key is examined at each step"; Eq. (1) weights).

    hist_fn(prefixes, prefix_bits, bits) -> [len(prefixes), 2^bits] GLOBAL (all-reduced)
    weights of the keys under each prefix.  Splitter j (1 <= j < K) is refined, `bits` key
    bits per round, down to the bin where the cumulative weight crosses j/K of the total,
    until that bin holds <= tol * total / K or the key is exhausted; rank j takes the keys
    >= splitter j.  Returns the K-1 splitter keys (uint64, non-decreasing)."""
    K = nranks
    if K <= 1:
        return np.zeros(0, dtype=np.uint64)
    h0 = np.asarray(hist_fn([0], 0, bits))[0]
    total = float(h0.sum())
    if total <= 0:
        return np.zeros(K - 1, dtype=np.uint64)
    b, resid = choose_bins(h0, total * np.arange(1, K) / K)
    prefix = [int(x) for x in b]
    weight = h0[b]
    pbits = bits
    while pbits < 63 and np.any(weight > tol * total / K):
        nb = min(bits, 63 - pbits)
        hs = np.asarray(hist_fn(prefix, pbits, nb))
        for j in range(K - 1):
            bj, rj = choose_bins(hs[j], resid[j:j + 1])
            prefix[j] = (prefix[j] << nb) | int(bj[0])
            resid[j] = rj[0]
            weight[j] = hs[j][bj[0]]
        pbits += nb
    out = np.array([p << (63 - pbits) for p in prefix], dtype=np.uint64)
    return np.maximum.accumulate(out)


COORD_BITS = 21   # R3 quantised coordinates


def orb_plan(hist_fn, split_fn, nranks: int, bits: int = 16):
    """ORB multisection for any rank count.

    Group ids are the first rank of the group's rank range, so after the last round a
    particle's group is its rank.  Every round, each group of Kg > 1 ranks is cut along the
    longest axis of its box (quantised coordinates, ties to the lower axis) where the global
    weight fraction reaches floor(Kg/2)/Kg; the cut coordinate is refined `bits` then the
    remaining bits (the same histogram refinement as partition_splitters) and particles with
    coordinate >= cut take the right half's id.
      hist_fn(axis[K], prefix[K], prefix_bits, bits) -> [K, 2^bits] global weights
      split_fn(axis[K], cut[K], right[K])
    Returns the list of groups {r0, r1, lo, hi} (boxes in quantised coordinates)."""
    K = nranks
    full = 1 << COORD_BITS
    groups = {0: dict(r0=0, r1=K, lo=[0, 0, 0], hi=[full, full, full])}
    while any(g["r1"] - g["r0"] > 1 for g in groups.values()):
        axis = np.full(K, -1, np.int32)
        frac = np.zeros(K)
        for gid, g in groups.items():
            if g["r1"] - g["r0"] > 1:
                ext = [g["hi"][a] - g["lo"][a] for a in range(3)]
                axis[gid] = int(np.argmax(ext))
                frac[gid] = ((g["r1"] - g["r0"]) // 2) / (g["r1"] - g["r0"])
        prefix = np.zeros(K, np.uint32)
        h = np.asarray(hist_fn(axis, prefix, 0, bits))
        total = h.sum(axis=1)
        resid = total * frac
        for gid in groups:
            if axis[gid] >= 0:
                b, r = choose_bins(h[gid], resid[gid:gid + 1]) if total[gid] > 0 else (np.array([0]), np.array([0.0]))
                prefix[gid] = int(b[0])
                resid[gid] = r[0]
        nb = COORD_BITS - bits
        h2 = np.asarray(hist_fn(axis, prefix, bits, nb))
        cut = np.zeros(K, np.uint32)
        right = np.zeros(K, np.int32)
        new = {}
        for gid, g in list(groups.items()):
            if axis[gid] < 0:
                new[gid] = g
                continue
            a = int(axis[gid])
            if total[gid] > 0:
                b2, _ = choose_bins(h2[gid], resid[gid:gid + 1])
                c = (int(prefix[gid]) << nb) | int(b2[0])
            else:
                c = (g["lo"][a] + g["hi"][a]) // 2
            c = min(max(c, g["lo"][a]), g["hi"][a])
            kl = (g["r1"] - g["r0"]) // 2
            rid = g["r0"] + kl
            cut[gid], right[gid] = c, rid
            lo_r, hi_l = list(g["lo"]), list(g["hi"])
            hi_l[a] = c
            lo_r[a] = c
            new[gid] = dict(r0=g["r0"], r1=rid, lo=g["lo"], hi=hi_l)
            new[rid] = dict(r0=rid, r1=g["r1"], lo=lo_r, hi=g["hi"])
        split_fn(axis, cut, right)
        groups = new
    return groups


# ------------------------------------------------------------------ Eq. (1) alpha over time steps
class AlphaTuner:
    """alpha of Eq. (1) w_i = l_i + alpha r_i, "a constant that is optimized over the time steps to
    minimize the total runtime" (§II-B; the paper names no method).  Reading: a
    golden-section search on log(alpha) over [lo, hi], one measured step runtime per probe, until
    the bracket is narrower than `tol` (in log alpha); then alpha stays at the fastest probe.

    The weights a step computes with alpha only shape the NEXT step's partition, so a probe is
    set for two consecutive steps and scored by the runtime of the second (the first step that
    ran on a partition made with it): next_alpha() before each step's weights, report(t) after
    each step."""

    GR = (np.sqrt(5.0) - 1.0) / 2.0

    def __init__(self, lo: float = 1.0 / 16, hi: float = 16.0, tol: float = 0.1):
        if not (0 < lo < hi):
            raise ValueError("need 0 < lo < hi")
        self.a, self.b, self.tol = float(np.log(lo)), float(np.log(hi)), tol
        self.c = self.b - self.GR * (self.b - self.a)
        self.d = self.a + self.GR * (self.b - self.a)
        self.fc = self.fd = None
        self.history = []            # (alpha, runtime) per scored probe
        self._probe = self.c         # log alpha being evaluated
        self._age = 0                # steps the current probe has been set for

    @property
    def converged(self) -> bool:
        return self.b - self.a < self.tol

    @property
    def best(self) -> float:
        if not self.history:
            return float(np.exp(self._probe))
        return min(self.history, key=lambda h: h[1])[0]

    def next_alpha(self) -> float:
        if self.converged:
            return self.best
        return float(np.exp(self._probe))

    def report(self, runtime: float) -> None:
        """runtime of the step just finished (its partition used the weights of the step before)."""
        if self.converged:
            return
        self._age += 1
        if self._age < 2:            # the probe's weights have not partitioned a step yet
            return
        self.history.append((float(np.exp(self._probe)), float(runtime)))
        if self._probe == self.c:
            self.fc = float(runtime)
        else:
            self.fd = float(runtime)
        if self.fc is None:
            self._probe = self.c
        elif self.fd is None:
            self._probe = self.d
        else:
            self._shrink()
        self._age = 0

    def _shrink(self) -> None:
        if self.fc < self.fd:        # minimum in [a, d]
            self.b, self.d, self.fd = self.d, self.c, self.fc
            self.c = self.b - self.GR * (self.b - self.a)
            self.fc = None
            self._probe = self.c
        else:                        # minimum in [c, b]
            self.a, self.c, self.fc = self.c, self.d, self.fd
            self.d = self.a + self.GR * (self.b - self.a)
            self.fd = None
            self._probe = self.d


# ------------------------------------------------------------------ driver
class DistFMM:
    """The FMM on `comm.world` ranks; this process drives the ranks `comm.ranks`.

    solve(pos[i], q[i], gid_base[i], w[i]) for every local rank i (device tensors of the
    contexts' precision) returns phi[i], grad[i] in the caller's particle order."""

    def __init__(self, comm: Comm, n_max: int, P: int, theta: float, ncrit: int, prec: str = "f32",
                 device: int = 0, hist_bits: int = HIST_BITS, alpha: float = 1.0, c_m2l: float = None,
                 partitioner: str = "morton"):
        if partitioner not in ("morton", "orb"):
            raise ValueError("partitioner must be 'morton' (Morton ranges) or 'orb' (multisection)")
        self.partitioner = partitioner
        self.comm, self.K = comm, comm.world
        self.fmm = [FMM(n_max, P, theta, ncrit, prec, device) for _ in comm.ranks]
        self.hist_bits = hist_bits
        self.alpha = alpha                                        # Eq. (1)
        self.c_m2l = m2l_cost_ratio(P) if c_m2l is None else c_m2l
        self.stats = {}
        self.weights = None                                       # per local rank, owner order
        self.tuner = None                                         # AlphaTuner (enable_alpha_tuning)

    def enable_alpha_tuning(self, lo: float = 1.0 / 16, hi: float = 16.0, tol: float = 0.1):
        """Optimise Eq. (1)'s alpha over the following solve(reuse_weights=True) steps by their
        measured runtime (max over ranks); see AlphaTuner."""
        self.tuner = AlphaTuner(lo, hi, tol)
        return self.tuner

    def close(self):
        for f in self.fmm:
            f.close()

    # 1-3: partition
    def partition(self, pos, q, gid_base, w=None):
        cm, K, F = self.comm, self.K, self.fmm
        nl = len(F)
        b = [torch.from_numpy(f.bounds(p)).to(p.device) for f, p in zip(F, pos)]
        lo = cm.allreduce([x[:3].clone() for x in b], "min")
        hi = cm.allreduce([x[3:].clone() for x in b], "max")
        gb = [torch.cat([lo[i], hi[i]]).cpu().numpy() for i in range(nl)]
        self.global_bounds = gb[0]
        keys = [F[i].part_keys(pos[i], gb[i]) for i in range(nl)]

        def hist_fn(prefixes, pbits, bits):
            loc = []
            for i in range(nl):
                h = torch.empty((len(prefixes), 1 << bits), dtype=torch.float64, device=keys[i].device)
                for r, pre in enumerate(prefixes):
                    F[i].part_histogram(keys[i], None if w is None else w[i], bits, pre, pbits, out=h[r])
                loc.append(h)
            return cm.allreduce(loc, "sum")[0].cpu().numpy()

        if self.partitioner == "morton":
            s = partition_splitters(hist_fn, K, self.hist_bits)
            packed = [F[i].part_pack(pos[i], q[i], keys[i], s, K, gid_base[i]) for i in range(nl)]
        else:
            grp = [torch.zeros(keys[i].shape[0], dtype=torch.int32, device=keys[i].device) for i in range(nl)]

            def orb_hist(axis, prefix, pbits, bits):
                loc = [F[i].orb_histogram(keys[i], grp[i], axis, prefix, pbits, bits,
                                          None if w is None else w[i]) for i in range(nl)]
                return cm.allreduce(loc, "sum")[0].cpu().numpy()

            def orb_split(axis, cut, right):
                for i in range(nl):
                    F[i].orb_split(keys[i], grp[i], axis, cut, right)

            self.orb_groups = orb_plan(orb_hist, orb_split, K, self.hist_bits)
            packed = [F[i].part_pack_dest(pos[i], q[i], grp[i], K, gid_base[i]) for i in range(nl)]
        cnt = [p[3] for p in packed]
        sp = cm.alltoallv([list(packed[i][0].reshape(-1).split((cnt[i] * 3).tolist())) for i in range(nl)])
        sq = cm.alltoallv([list(packed[i][1].split(cnt[i].tolist())) for i in range(nl)])
        sg = cm.alltoallv([list(packed[i][2].split(cnt[i].tolist())) for i in range(nl)])
        lpos = [torch.cat(sp[i]).reshape(-1, 3).contiguous() for i in range(nl)]
        lq = [torch.cat(sq[i]).contiguous() for i in range(nl)]
        lgid = [torch.cat(sg[i]) for i in range(nl)]
        back = [[int(t.numel()) for t in sq[i]] for i in range(nl)]   # segment sizes per source rank
        return lpos, lq, lgid, back, packed, cnt

    # 4-5: local trees, LET structure, traversal
    def build(self, lpos):
        cm, K, F = self.comm, self.K, self.fmm
        nl = len(F)
        dev = lpos[0].device
        for f, p in zip(F, lpos):
            # Morton ranges are pieces of the global curve: build each local tree on the global
            # root cube so it is a subtree of the global octree (no slivers at the range ends);
            # ORB boxes are compact: local bounding box
            f.set_root_bounds(self.global_bounds if self.partitioner == "morton" else None)
            f.build_tree(p)
        cov = []
        for f in F:
            c = f.let_cover()
            t = torch.zeros(1 + 8 * 73, dtype=torch.float64)
            t[0] = len(c)
            t[1:1 + c.size] = torch.from_numpy(c.reshape(-1))
            cov.append(t.to(dev))
        allcov = cm.allgather(cov)
        self._dbytes = []
        sends = []
        for i, f in enumerate(F):
            me = cm.ranks[i]
            row, db = [], []
            for j in range(K):
                if j == me:
                    row.append(torch.empty(0, dtype=torch.uint8, device=dev))
                    db.append(0)
                    continue
                cj = allcov[i][j].cpu().numpy()
                sb, d = f.let_plan(j, cj[1:1 + 8 * int(cj[0])].reshape(-1, 8))
                buf = torch.empty(sb, dtype=torch.uint8, device=dev)
                if sb:
                    f.let_pack_struct(j, buf)
                row.append(buf)
                db.append(d)
            sends.append(row)
            self._dbytes.append(db)
        # sizes first (one small all-to-all), then K-1 ring rounds: in round s every rank sends
        # its LET to rank me+s and receives rank me-s's.  Round s+1 is in flight while round
        # s's fragment is grafted and traversed (each message processed as it
        # lands); the local traversal overlaps round 1.
        szs = cm.alltoallv([[torch.tensor([t.numel()], dtype=torch.int64, device=dev) for t in row]
                            for row in sends])
        rsz = [[int(x) for x in torch.cat(szs[i]).tolist()] for i in range(nl)]
        me = cm.ranks

        def start(sr):
            dst = [(me[i] + sr) % K for i in range(nl)]
            src = [(me[i] - sr) % K for i in range(nl)]
            return cm.sendrecv([sends[i][dst[i]] for i in range(nl)], dst, src,
                               [rsz[i][src[i]] for i in range(nl)], async_op=True), src

        self._peers = [[] for _ in range(nl)]
        h = start(1) if K > 1 else None
        for f in F:                       # local traversal overlaps the first LET round
            f.dtt(remote=False)
        for sr in range(1, K):
            hh, src = h
            recv = hh.wait()
            if sr + 1 < K:
                h = start(sr + 1)
            for i, f in enumerate(F):
                if recv[i].numel() > 0:
                    f.let_graft([recv[i]])
                    f.dtt(remote=True)    # traverses only the fragment just grafted
                    self._peers[i].append(src[i])
        for f in F:
            f.make_lists()
        self.stats["let_struct_bytes"] = sum(int(t.numel()) for row in sends for t in row)

    # 6: upward, LET data, interactions
    def evaluate(self, lpos, lq):
        cm, K, F = self.comm, self.K, self.fmm
        dev = lpos[0].device
        sends = []
        for i, f in enumerate(F):
            f.upward(lpos[i], lq[i])
            me = cm.ranks[i]
            row = []
            for j in range(K):
                d = self._dbytes[i][j]
                buf = torch.empty(d, dtype=torch.uint8, device=dev)
                if d and j != me:
                    f.let_pack_data(j, buf)
                row.append(buf)
            sends.append(row)
        recv = cm.alltoallv(sends)
        out = []
        for i, f in enumerate(F):
            f.let_unpack([recv[i][j] for j in self._peers[i]])    # graft (ring) order
            n = lpos[i].shape[0]
            phi = torch.empty(n, dtype=f.dtype, device=dev)
            grad = torch.empty((n, 3), dtype=f.dtype, device=dev)
            f.interact(phi, grad)
            out.append((phi, grad))
        self.stats["let_data_bytes"] = sum(int(t.numel()) for row in sends for t in row)
        return out

    # 4-6 in one pass (solve): the upward pass runs on a side stream while the covers are
    # exchanged, the LET structures planned and the local tree traversed, so each ring message
    # carries structure AND data (one exchange instead of two) and every fragment is grafted,
    # unpacked and traversed as it lands (round s+1 in flight meanwhile)
    def build_evaluate(self, lpos, lq):
        cm, K, F = self.comm, self.K, self.fmm
        nl = len(F)
        dev = lpos[0].device
        main = torch.cuda.current_stream(dev)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(dev)
        side = self._side
        for f, p in zip(F, lpos):
            f.set_root_bounds(self.global_bounds if self.partitioner == "morton" else None)
            f.build_tree(p)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            for i, f in enumerate(F):
                f.upward(lpos[i], lq[i], stream=side)
        up_done = side.record_event()
        cov = []
        for f in F:
            c = f.let_cover()
            t = torch.zeros(1 + 8 * 73, dtype=torch.float64)
            t[0] = len(c)
            t[1:1 + c.size] = torch.from_numpy(c.reshape(-1))
            cov.append(t.to(dev))
        allcov = cm.allgather(cov)
        plans, sends = [], []
        for i, f in enumerate(F):
            me = cm.ranks[i]
            row, pl = [], []
            for j in range(K):
                if j == me:
                    row.append(torch.empty(0, dtype=torch.uint8, device=dev))
                    pl.append((0, 0))
                    continue
                cj = allcov[i][j].cpu().numpy()
                sb, d = f.let_plan(j, cj[1:1 + 8 * int(cj[0])].reshape(-1, 8))
                buf = torch.empty(sb + d, dtype=torch.uint8, device=dev)   # [structure | data]
                if sb:
                    f.let_pack_struct(j, buf[:sb])
                row.append(buf)
                pl.append((sb, d))
            sends.append(row)
            plans.append(pl)
        for f in F:                       # local traversal overlaps the side-stream upward pass
            f.dtt(remote=False)
        main.wait_event(up_done)
        for i, f in enumerate(F):
            me = cm.ranks[i]
            for j in range(K):
                sb, d = plans[i][j]
                if d and j != me:
                    f.let_pack_data(j, sends[i][j][sb:])
        szs = cm.alltoallv([[torch.tensor(list(plans[i][j]), dtype=torch.int64, device=dev) for j in range(K)]
                            for i in range(nl)])
        rsz = [[tuple(int(x) for x in t.tolist()) for t in szs[i]] for i in range(nl)]
        me = cm.ranks

        def start(sr):
            dst = [(me[i] + sr) % K for i in range(nl)]
            src = [(me[i] - sr) % K for i in range(nl)]
            return cm.sendrecv([sends[i][dst[i]] for i in range(nl)], dst, src,
                               [sum(rsz[i][src[i]]) for i in range(nl)], async_op=True), src

        self._peers = [[] for _ in range(nl)]
        h = start(1) if K > 1 else None
        for sr in range(1, K):
            hh, src = h
            recv = hh.wait()
            if sr + 1 < K:
                h = start(sr + 1)
            for i, f in enumerate(F):
                rsb, _ = rsz[i][src[i]]
                if rsb > 0:
                    f.let_graft([recv[i][:rsb]])
                    f.let_unpack([recv[i][rsb:]], first=len(self._peers[i]))
                    f.dtt(remote=True)    # traverses only the fragment just grafted
                    self._peers[i].append(src[i])
        out = []
        for i, f in enumerate(F):
            f.make_lists()
            n = lpos[i].shape[0]
            phi = torch.empty(n, dtype=f.dtype, device=dev)
            grad = torch.empty((n, 3), dtype=f.dtype, device=dev)
            f.interact(phi, grad)
            out.append((phi, grad))
        self.stats["let_struct_bytes"] = sum(p[0] for pl in plans for p in pl)
        self.stats["let_data_bytes"] = sum(p[1] for pl in plans for p in pl)
        return out

    # 7: results (and the Eq. (1) weights of this step) back to the owners, original order
    def gather_back(self, res, wts, back, packed, cnt, gid_base, n_in):
        cm = self.comm
        nl = len(self.fmm)
        sends = []
        for i in range(nl):
            phi, grad = res[i]
            v = torch.cat([phi.reshape(-1, 1), grad, wts[i].to(phi.dtype).reshape(-1, 1)], dim=1)   # [n, 5]
            sends.append(list(v.reshape(-1).split([5 * s for s in back[i]])))
        recv = cm.alltoallv(sends)
        out, wout = [], []
        for i in range(nl):
            v = torch.cat(recv[i]).reshape(-1, 5)              # in this rank's packed order
            idx = packed[i][2] - gid_base[i]                    # original local index
            r = torch.empty((n_in[i], 5), dtype=v.dtype, device=v.device)
            r[idx] = v
            out.append((r[:, 0].contiguous(), r[:, 1:4].contiguous()))
            wout.append(r[:, 4].float().contiguous())
        return out, wout

    def solve(self, pos, q, gid_base, w=None, reuse_weights=False):
        """One distributed FMM step.  w: per-rank particle weights for the partition (None:
        1, or with reuse_weights the Eq. (1) weights this object measured at its last step)."""
        if w is None and reuse_weights and self.weights is not None:
            w = self.weights
        if self.tuner is not None:
            dev = pos[0].device
            if dev.type == "cuda":
                torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            self.alpha = self.tuner.next_alpha()                 # for this step's weights
        lpos, lq, lgid, back, packed, cnt = self.partition(pos, q, gid_base, w)
        res = self.build_evaluate(lpos, lq)
        wts = []
        lr = np.zeros(2)
        for f in self.fmm:
            wi, s = f.work(self.c_m2l, self.alpha)
            wts.append(wi)
            lr += s
        self.stats["work_local"], self.stats["work_remote"] = float(lr[0]), float(lr[1])
        self.local = (lpos, lq, lgid)
        out, self.weights = self.gather_back(res, wts, back, packed, cnt, gid_base, [p.shape[0] for p in pos])
        if self.tuner is not None:
            if dev.type == "cuda":
                torch.cuda.synchronize(dev)
            t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            t = self.comm.allreduce([t] * len(self.fmm), "max")[0]
            self.tuner.report(float(t.item()))
            self.stats["alpha"] = self.alpha
        return out
