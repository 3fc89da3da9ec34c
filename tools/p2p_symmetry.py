"""Symmetry of the P2P leaf-pair lists: entries (A, B) whose mirror (B, A) is also listed, and their
share of the body-body interactions (mutual P2P analysis)."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, synth
from paper_1405_7487_b200.fmm import FMM
for name in ["c2", "sph", "c3"]:
    c = synth.CONFIGS[name]
    pos, _ = synth.generate(c["kind"], c["n"], c["seed"], np.float32)
    f = FMM(c["n"], c["P"], c["theta"], c["ncrit"], c["prec"])
    f.build(torch.from_numpy(pos).cuda()); torch.cuda.synchronize()
    _, p2p = f.lists()
    a = p2p[:, 0].astype(np.uint64); b = p2p[:, 1].astype(np.uint64)
    k = np.sort((a << np.uint64(32)) | b); km = np.sort((b << np.uint64(32)) | a)
    sym = np.isin(k, km, assume_unique=True)
    cells = f.cells(); bc = cells["body_count"].astype(np.int64)
    w = bc[p2p[:, 0]] * bc[p2p[:, 1]]
    self_ = a == b
    print(name, "entries", len(a), "self", int(self_.sum()), "symmetric", int(sym.sum()), "asym", int((~sym).sum()),
          "interactions sym-nonself share", float(w[(~self_) & np.isin((a << np.uint64(32)) | b, km)].sum() / w.sum()))
    f.close()
