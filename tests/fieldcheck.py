"""Field comparison used by every GPU-vs-oracle test.

Two bounds, both against the oracle b (north_star tolerances):
  * relative L2  ||a - b||_2 / ||b||_2 <= tol  (over all values of phi, or all 3n gradient components);
  * per-element  max_i |a_i - b_i| / max_i |b_i| <= 10 tol, so that one wrong target (or one
    wrong leaf) cannot hide under a global norm: at N = 2^20 one target off by 1e-4 gives a
    relative L2 of ~3e-6, which the L2 bound alone would accept.
"""
import numpy as np

import oracle


def field_errors(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    scale = np.abs(b).max() if b.size else 0.0
    emax = float(np.abs(a - b).max() / scale) if b.size and scale > 0 else float(np.abs(a - b).max(initial=0.0))
    return oracle.rel_l2(a, b), emax


def assert_field(a, b, tol, what=""):
    l2, emax = field_errors(a, b)
    assert l2 <= tol, f"{what}: relative L2 {l2:.3e} > {tol:.1e}"
    assert emax <= 10 * tol, f"{what}: max |diff| / max |ref| {emax:.3e} > {10 * tol:.1e}"
    return l2, emax


def assert_fields(phi, ophi, grad, ograd, tol, what=""):
    e1 = assert_field(phi, ophi, tol, f"{what} phi")
    e2 = assert_field(grad, ograd, tol, f"{what} grad")
    return e1, e2
