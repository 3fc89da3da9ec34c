#!/usr/bin/env python
"""bench.py -- FMM particles/s on B200 (BASELINE.json metric), one JSON line on rank 0.

Step = one pass of the whole hot path on one synthetic input:
fmm_build (bounds, keys, radix sort, octree, geometry, dual tree traversal, lists) +
fmm_evaluate (P2M/M2M, M2L, P2P, L2L/L2P, un-permute), inputs resident in HBM.
Default workload: BASELINE.json configs[1] (N = 2^20 uniform cube, fp32, P=10, theta=0.4,
ncrit=64).  L2 is flushed (256 MB write) before every timed step; each step is timed with
CUDA events on the stream the library runs on.

  python bench.py [--gpus N --steps K --warmup W] [--config c2|c3|c1] [--impl reference]

Multi-GPU (torchrun, --gpus N > 1): ONE FMM over N x 2^20 particles (weak scaling: each rank
starts with its 2^20-particle slice of one global cube set), solved by the distributed path
(paper_1405_7487_b200/dist.py over NCCL): Morton-range partition, local trees, LET exchange
overlapped with the local traversal, remote traversal, M2L/P2P, results back to the owners.
Step time = max over ranks of the CUDA-event time around the whole distributed solve; every
step partitions with the Eq. (1) weights measured in the previous step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "FMM particles/s at 1/2/4/8 B200 (P=10); P2P+M2L % of FP32 roofline"
CONFIG_NAMES = {"c1": "configs[0]", "c2": "configs[1]", "c3": "configs[2]", "sph": "Table I case 2 (sphere)",
                "c4s": "configs[3] (strong-scaling N on 1 GPU)", "c4w": "configs[3] (weak-scaling per-GPU N)"}
FP32_LANES_PER_SM = 128


# ----------------------------------------------------------- algorithmic work
from paper_1405_7487_b200.costs import P2P_FLOPS, P2P_INSTR, m2l_flops_per_pair, t2n  # noqa: E402,F401


def peaks():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        return json.load(f)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ oracle (CPU) arm
def oracle_rate(cfg: dict, n_sample: int, reps: int = 1):
    """The CPU oracle as it stands: full FMM on a bounded sample of the workload (same
    distribution, P, theta, ncrit; first n_sample particles of a seed-identical draw)."""
    import oracle
    oracle.build()
    dt = np.float32 if cfg["prec"] == "f32" else np.float64
    pos, q = synth.generate(cfg["kind"], n_sample, cfg["seed"], dt)
    p64, q64 = pos.astype(np.float64), q.astype(np.float64)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        o = oracle.FMM(p64, q64, cfg["P"], cfg["theta"], cfg["ncrit"])
        o.evaluate()
        times.append(time.perf_counter() - t0)
        del o
    return n_sample, times


def host_cpu():
    """Host CPU model and logical core count (lscpu / os.cpu_count) for the oracle's baseline."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.TimeoutExpired):
        pass
    return {"model": model, "nproc": os.cpu_count()}


def cpu_baseline(cfg):
    n_s = 1 << 14
    n, times = oracle_rate(cfg, n_s)
    return {"value": n / times[0], "unit": "particles/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
            "sample": f"full oracle FMM (keys..L2P) on {n} particles of the {cfg['kind']} distribution with the "
                      f"workload's P={cfg['P']}, theta={cfg['theta']}, ncrit={cfg['ncrit']}; single-threaded fp64 "
                      f"C, {times[0]:.1f} s"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle on the host cores, same metric/unit (rank 0 only)."""
    if rank != 0:
        return
    n_s = 1 << 13
    n, times = oracle_rate(cfg, n_s, reps=args.warmup + args.steps)
    timed = times[args.warmup:]
    t = sum(timed) / len(timed)
    line = {"metric": METRIC, "impl": "reference", "value": n / t, "unit": "particles/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args, world),
            "cpu_baseline": {"value": n / t, "unit": "particles/s", "cores": 1, "kind": "oracle", "host": host_cpu(),
                             "sample": f"full oracle FMM on {n} particles of the workload's distribution and "
                                       f"parameters per step"},
            "e2e": {"value": n / t, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(cfg, args, world=1, N=None):
    n = cfg["n"] * world if N is None else N
    d = {"workload": f"BASELINE.json {CONFIG_NAMES[args.config]}: 3D Laplace FMM, N={n} {cfg['kind']}, "
                     f"{cfg['prec']}, P={cfg['P']}, theta={cfg['theta']}, ncrit={cfg['ncrit']}",
         "N": n, "distribution": cfg["kind"], "P": cfg["P"], "theta": cfg["theta"], "ncrit": cfg["ncrit"],
         "precision": cfg["prec"], "seed": cfg["seed"], "l2": "flushed (256 MB write) before every timed step",
         "parallelism": "1 GPU"}
    if world > 1 or getattr(args, "dist", False):
        part = "ORB multisection" if getattr(args, "partitioner", "morton") == "orb" else "Morton-range"
        how = (f"weak scaling at constant density, {cfg['n']} particles per GPU, rank r's particles in unit cube r "
               f"of a 2x2x2 Morton block pattern" if args.scaling == "weak" else
               f"strong scaling, one {cfg['n']}-particle set split into {world} index slices")
        d["parallelism"] = (f"{world} GPU(s), one FMM through fmm_dist_solve: {part} partition with Eq. (1) weights + "
                            f"LET exchange over NCCL ({how})")
        d["workload"] = (f"BASELINE.json configs[3] ({args.scaling} scaling, " + CONFIG_NAMES[args.config] +
                         f"): 3D Laplace FMM, N={n} {cfg['kind']}, {cfg['prec']}, P={cfg['P']}, theta={cfg['theta']}, "
                         f"ncrit={cfg['ncrit']}")
        d["scaling"] = args.scaling
    return d


def roofline_block(args, cfg, counts, ph):
    """Dominant kernel against the FP32 ALU peak.  `achieved` counts
    algorithmic flops (P2P: 18 per interaction, FFMA = 2; M2L: the harmonic form's FMA + recurrence
    ops, costs.py); P2P's primary figure, the FP32 issue-slot fraction (13 lane-ops per interaction),
    is reported beside it as `fp32_issue_frac`."""
    pk = peaks()
    sm_mhz = pk["sm_max_mhz"]
    fp32_peak_tflops = 148 * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12     # FFMA = 2 flops
    lane_peak = 148 * FP32_LANES_PER_SM * sm_mhz * 1e6                         # lane-ops/s
    m2l = m2l_flops_per_pair(cfg["P"])
    m2l_ms = ph.get("m2l_kernel", 0.0) / args.steps
    p2p_ms = ph.get("p2p_kernel", 0.0) / args.steps
    m2l_tf = counts["n_m2l"] * m2l["flops"] / (m2l_ms * 1e-3) / 1e12 if m2l_ms else 0.0
    p2p_tf = counts["p2p_interactions"] * P2P_FLOPS / (p2p_ms * 1e-3) / 1e12 if p2p_ms else 0.0
    p2p_issue = counts["p2p_interactions"] * P2P_INSTR / (p2p_ms * 1e-3) / lane_peak if p2p_ms else None
    m2l_issue = counts["n_m2l"] * m2l["instr"] / (m2l_ms * 1e-3) / lane_peak if m2l_ms else None
    dom = "m2l" if m2l_ms >= p2p_ms else "p2p"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"{args.config}:{dom}")
    ach = m2l_tf if dom == "m2l" else p2p_tf
    return {"kernel": f"{dom} ({'k_m2l_mir' if dom == 'm2l' else 'k_p2p_tma + k_p2p_cta (leaf classes)'})",
            "bound": "alu", "achieved": round(ach, 3), "peak": round(fp32_peak_tflops, 2),
            "unit": "TFLOP/s", "frac": round(ach / fp32_peak_tflops, 4), "traffic": traffic,
            "fp32_issue_frac": round((m2l_issue if dom == "m2l" else p2p_issue) or 0.0, 4),
            "flops_per_unit": m2l["flops"] if dom == "m2l" else P2P_FLOPS,
            "units_per_launch": counts["n_m2l"] if dom == "m2l" else counts["p2p_interactions"],
            "peak_note": "FP32 FFMA peak = 148 SMs x 128 lanes x 2 flop x sm_max_mhz (MEASURED_PEAKS.json); "
                         "fp32_issue_frac = lane-ops per unit (P2P 13, SURVEY §8(d) item 1) x units/s / "
                         "(148 x 128 x sm_max_mhz); DESIGN.md §6",
            "per_kernel": {
                "m2l": {"ms": round(m2l_ms, 4), "pairs": counts["n_m2l"], "flops_per_pair": m2l["flops"],
                        "instr_per_pair": m2l["instr"], "TFLOP/s": round(m2l_tf, 3),
                        "frac": round(m2l_tf / fp32_peak_tflops, 4),
                        "fp32_issue_frac": round(m2l_issue, 4) if m2l_issue else None,
                        "pairs_per_s": counts["n_m2l"] / (m2l_ms * 1e-3) if m2l_ms else None},
                "p2p": {"ms": round(p2p_ms, 4), "interactions": counts["p2p_interactions"],
                        "flops_per_interaction": P2P_FLOPS, "instr_per_interaction": P2P_INSTR,
                        "TFLOP/s": round(p2p_tf, 3), "frac": round(p2p_tf / fp32_peak_tflops, 4),
                        "fp32_issue_frac": round(p2p_issue, 4) if p2p_issue else None,
                        "interactions_per_s": counts["p2p_interactions"] / (p2p_ms * 1e-3) if p2p_ms else None}},
            "measured": "CUDA events recorded by libfmm around each kernel on the stream it runs on (P2P then "
                        "M2L, back to back on the caller's stream); per-launch average over the timed steps",
            "traffic_note": "dram read+write bytes per launch from one ncu --set full capture (profiles/traffic.json)"}


def weak_offset(r: int) -> np.ndarray:
    """Weak scaling at constant density: rank r's particles fill unit cube r of a block pattern in
    Morton order (r bits -> x, y, z, x, ...; 2 GPUs: 2x1x1, 4: 2x2x1, 8: 2x2x2), so every GPU's
    particles have the same spacing and its tree the same leaf occupancy as the 1-GPU case."""
    o = np.zeros(3)
    for b in range(max(r.bit_length(), 1)):
        o[b % 3] += ((r >> b) & 1) << (b // 3)
    return o


def dist_input(cfg, scaling, rank, world):
    """(pos, q, gid_base, N_total) of this rank.  weak: cfg['n'] particles per rank in rank r's unit
    cube (constant density); strong: rank r's contiguous slice of ONE cfg['n']-particle set."""
    dt_np = np.float32 if cfg["prec"] == "f32" else np.float64
    if scaling == "weak":
        n = cfg["n"]
        pos, q = synth.generate(cfg["kind"], n, cfg["seed"], dt_np, start=rank * n, n_total=n * world)
        return (pos + weak_offset(rank)).astype(dt_np), q, rank * n, n * world
    N = cfg["n"]
    lo, hi = rank * N // world, (rank + 1) * N // world
    pos, q = synth.generate(cfg["kind"], hi - lo, cfg["seed"], dt_np, start=lo, n_total=N)
    return pos, q, lo, N


def run_dist(args, cfg, rank, world, local):
    """--gpus N > 1 under torchrun (or --dist on one GPU): the library's distributed driver
    (fmm_create_dist / fmm_dist_solve over NCCL; the process group only broadcasts the NCCL id and
    times the step as the max over ranks)."""
    import torch
    import torch.distributed as tdist
    from paper_1405_7487_b200.dist import DistFMM, nccl_unique_id
    dt_t = torch.float32 if cfg["prec"] == "f32" else torch.float64
    pos, q, gid_base, N = dist_input(cfg, args.scaling, rank, world)
    n = len(pos)
    dpos = torch.from_numpy(pos).cuda()
    dq = torch.from_numpy(q).cuda()
    uid = [nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(uid, src=0)
    # a rank may own up to twice its share after an Eq. (1)-weighted partition
    D = DistFMM(max(2 * N // world, n) + 1024, cfg["P"], cfg["theta"], cfg["ncrit"], cfg["prec"], local, world, rank,
                unique_id=uid[0], partitioner=args.partitioner)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    phi = torch.empty(n, dtype=dt_t, device="cuda")
    grad = torch.empty((n, 3), dtype=dt_t, device="cuda")

    def step():
        # every step after the first partitions with the previous step's Eq. (1) weights
        D.solve(dpos, dq, gid_base, reuse_weights=True, phi=phi, grad=grad, stream=stream)

    if args.tune_alpha > 0:
        # Eq. (1) alpha optimised over time steps before the measured run, then frozen
        D.tune_alpha()
        for _ in range(args.tune_alpha):
            step()
        D.tune_alpha(0.0, 0.0, 0.0)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    D.set_timing(True)
    D.phase_times(reset=True)
    D.launch_count(reset=True)
    tdist.barrier()
    torch.cuda.synchronize()
    ms = 0.0
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            b.synchronize()
            ms += a.elapsed_time(b)
        tdist.barrier()
        torch.cuda.synchronize()
    launches = D.launch_count(reset=True)
    ph = D.phase_times(reset=True)
    timeline = D.timeline()
    D.set_timing(False)
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    # e2e: pinned host buffers in, host results out, copies inside the timed region
    hpos = torch.from_numpy(pos).pin_memory()
    hq = torch.from_numpy(q).pin_memory()
    hphi = torch.empty(n, dtype=dt_t).pin_memory()
    hgrad = torch.empty((n, 3), dtype=dt_t).pin_memory()
    tdist.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(3, args.steps // 2)
    for _ in range(e2e_steps):
        gp = hpos.to("cuda", non_blocking=True)
        gq = hq.to("cuda", non_blocking=True)
        p_, g_ = D.solve(gp, gq, gid_base, reuse_weights=True, stream=stream)
        hphi.copy_(p_, non_blocking=True)
        hgrad.copy_(g_, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    e2e_s = float(t.item())
    counts = D.counts()
    st = D.stats()
    es = 4 if cfg["prec"] == "f32" else 8
    if rank == 0:
        line = {"metric": METRIC, "value": N / (ms_step * 1e-3), "unit": "particles/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f32" if cfg["prec"] == "f32" else "f64",
                "data": "synthetic (seeded SplitMix64 generator, synth/; each rank draws its slice)",
                "config": workload_config(cfg, args, world, N),
                "e2e": {"value": N / e2e_s, "unit": "particles/s", "h2d_bytes_per_step": n * 4 * es,
                        "d2h_bytes_per_step": n * 4 * es, "api": "fmm_dist_solve (pinned host buffers, per rank)"},
                "gpu_launches": launches,
                "roofline": roofline_block(args, cfg, counts, ph),
                "clocks": clk.summary(),
                "phases_ms": {k: round(v / args.steps, 4) for k, v in ph.items()},
                "timeline_ms_rank0": {k: [round(x, 3) for x in v] for k, v in timeline.items()},
                "phases_note": "per-phase CUDA-event spans; upward overlaps dtt/lists and downward overlaps p2p "
                               "(aux stream), so the spans sum to more than ms_per_step",
                "counts_rank0": counts,
                "dist_rank0": {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in st.items()},
                "alpha_tuned_steps": args.tune_alpha}
        print(json.dumps(line), flush=True)
    tdist.barrier()
    D.close()


# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIG_NAMES),
                    help="default: c2 on 1 GPU; with --gpus N > 1 (or --dist): c4w (weak) / c4s (strong)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="multi-GPU: weak = the config's N per GPU (BASELINE configs[3]: 2^24), strong = the "
                         "config's N in total (configs[3]: 2^26)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true", help="use the distributed path even on 1 GPU")
    ap.add_argument("--tune-alpha", type=int, default=0,
                    help="distributed path: optimise Eq. (1)'s alpha over this many steps before the warm-up")
    ap.add_argument("--partitioner", default="morton", choices=["morton", "orb"],
                    help="multi-GPU partition: Morton ranges (north_star) or ORB multisection (SURVEY 8f f3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = "c2" if world == 1 and not args.dist else ("c4w" if args.scaling == "weak" else "c4s")
    cfg = synth.CONFIGS[args.config]

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    from paper_1405_7487_b200 import FMM, build
    build.build()
    dist = None
    if world > 1 or args.dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
        run_dist(args, cfg, rank, world, local)
        dist.destroy_process_group()
        return
    dt_np = np.float32 if cfg["prec"] == "f32" else np.float64
    dt_t = torch.float32 if cfg["prec"] == "f32" else torch.float64
    n = cfg["n"]
    pos, q = synth.generate(cfg["kind"], n, cfg["seed"] + rank, dt_np)
    dpos = torch.from_numpy(pos).cuda()
    dq = torch.from_numpy(q).cuda()
    phi = torch.empty(n, dtype=dt_t, device="cuda")
    grad = torch.empty((n, 3), dtype=dt_t, device="cuda")
    fmm = FMM(n, cfg["P"], cfg["theta"], cfg["ncrit"], cfg["prec"], local)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2

    def step():
        fmm.solve(dpos, dq, phi, grad, stream)   # fmm_solve = fmm_build + fmm_evaluate, overlapped

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    fmm.set_timing(True)
    fmm.phase_times(reset=True)
    fmm.launch_count(reset=True)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        barrier()
    launches = fmm.launch_count(reset=True)
    ph = fmm.phase_times(reset=True)
    fmm.set_timing(False)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * n / (ms_step * 1e-3)

    # ---- e2e: host buffers through fmm_solve_host (H2D + D2H inside the timed region)
    hpos = torch.from_numpy(pos).pin_memory().numpy()
    hq = torch.from_numpy(q).pin_memory().numpy()
    hphi = torch.empty(n, dtype=dt_t).pin_memory().numpy()
    hgrad = torch.empty((n, 3), dtype=dt_t).pin_memory().numpy()
    fmm.solve_host(hpos, hq, hphi, hgrad)
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(3, args.steps // 2)
    for _ in range(e2e_steps):
        flush.fill_(0.0)
        torch.cuda.synchronize()
        fmm.solve_host(hpos, hq, hphi, hgrad)      # synchronous: returns after the D2H copy
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    es = 4 if cfg["prec"] == "f32" else 8

    counts = fmm.counts()
    if rank == 0:
        clocks = clk.summary()
        roof = roofline_block(args, cfg, counts, ph)
        line = {"metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32" if cfg["prec"] == "f32" else "f64",
                "data": "synthetic (seeded SplitMix64 generator, synth/)",
                "config": workload_config(cfg, args),
                "e2e": {"value": world * n / e2e_s, "unit": "particles/s", "h2d_bytes_per_step": n * 4 * es,
                        "d2h_bytes_per_step": n * 4 * es, "api": "fmm_solve_host (pinned host buffers)"},
                "gpu_launches": launches,
                "roofline": roof,
                "clocks": clocks,
                "phases_ms": {k: round(v / args.steps, 4) for k, v in ph.items()},
                "phases_note": "per-phase CUDA-event spans; upward overlaps dtt/lists and downward overlaps p2p "
                               "(aux stream), so the spans sum to more than ms_per_step",
                "counts": counts}
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
