"""Shared test helpers: seeded inputs from the workload module, oracle side setup."""
import numpy as np

from paper_1412_3784_b200 import workloads as W


def inputs(k, prec="f64", scale=1, r=0, flow="uniaxial"):
    """Workload C<k> (scaled) and its positions in storage precision."""
    w = W.make(k, r, flow=flow, scale=scale)
    dt = np.float32 if prec == "f32" else np.float64
    q = W.positions(w, dtype=dt, k=k, r=r)
    return w, q


def oracle_side(q, L, prec):
    """What the oracle consumes: the same stored values, wrapped by its own rule."""
    import oracle

    return oracle.wrap(np.asarray(q, dtype=np.float64), L, prec)
