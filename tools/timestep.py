"""Multi-step use of the distributed FMM: a leapfrog N-body integration where every
step re-partitions with the previous step's Eq. (1) weights and Eq. (1)'s alpha is optimised over
the steps by measured runtime (fmm_dist_tune_alpha).  Gravity with G = 1: masses are the charges,
the acceleration is +grad(phi) of phi = sum m_j / r (the library's sign), and the energy
E = sum m v^2 / 2 - sum m phi / 2 is printed so the drift can be checked.

    python tools/timestep.py [K ranks (an in-process group on one GPU)] [N] [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1405_7487_b200.dist import DistFMM, LocalGroup, run_ranks  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 17
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    pos, m = synth.generate("plummer", n, 7, np.float64)
    m = np.full(n, 1.0 / n)
    rng = np.random.default_rng(7)
    vel = rng.normal(scale=0.3, size=(n, 3))          # a warm start; any velocities do
    vel -= vel.mean(0)
    cuts = np.linspace(0, n, K + 1).astype(int)
    G = LocalGroup(K)
    D = [DistFMM(n, 6, 0.5, 32, "f64", 0, K, r, group=G) for r in range(K)]
    for f in D:
        f.tune_alpha(0.25, 4.0, 0.3)
    streams = [torch.cuda.Stream() for _ in range(K)]
    dt = 1e-3

    def forces(p):
        P_in = [torch.from_numpy(np.ascontiguousarray(p[cuts[r]:cuts[r + 1]])).cuda() for r in range(K)]
        M_in = [torch.from_numpy(np.ascontiguousarray(m[cuts[r]:cuts[r + 1]])).cuda() for r in range(K)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = run_ranks(lambda r: D[r].solve(P_in[r], M_in[r], int(cuts[r]), reuse_weights=True,
                                             stream=streams[r]), K)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        phi = np.concatenate([o[0].cpu().numpy() for o in out])
        acc = np.concatenate([o[1].cpu().numpy() for o in out])
        return phi, acc, t

    phi, acc, _ = forces(pos)
    e0 = 0.5 * np.sum(m * np.sum(vel ** 2, 1)) - 0.5 * np.sum(m * phi)
    for k in range(steps):
        vel += 0.5 * dt * acc
        pos += dt * vel
        phi, acc, t = forces(pos)
        vel += 0.5 * dt * acc
        e = 0.5 * np.sum(m * np.sum(vel ** 2, 1)) - 0.5 * np.sum(m * phi)
        st = D[0].stats()
        print(f"step {k:3d}  {1e3 * t:7.2f} ms  alpha {st['alpha']:6.3f}  work l/r {st['work_local']:.3e}/"
              f"{st['work_remote']:.3e}  dE/E {abs(e - e0) / abs(e0):.2e}", flush=True)
    st = D[0].stats()
    print("alpha probes", st["tuner_probes"], "best", round(st["tuner_best"], 3), "converged", st["tuner_converged"])
    for f in D:
        f.close()
    G.close()


if __name__ == "__main__":
    main()
