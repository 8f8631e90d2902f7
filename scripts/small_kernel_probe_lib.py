"""The paper's E2 system (scripts/e2_runtime.py's construction) for the small-system probes."""
import numpy as np

from paper_1412_3784_b200 import workloads as W


def e2():
    K = 12
    n = K ** 3
    a = (n / W.RHO) ** (1.0 / 3.0)
    M1, M2, L0, om1, om2 = W.gkr_params(a)
    adiag = np.array([2.0, -1.0, -1.0])
    eps = 0.025
    A = np.diag(eps * adiag)
    beta = np.linalg.lstsq(np.stack([om1, om2], axis=1), adiag, rcond=None)[0]
    extra = {"beta": beta, "eps": eps, "om1": om1, "om2": om2}
    L = W.box_at(L0, A, "gkr", 0.0, extra)
    return W.Workload("E2", n, L0, A, "gkr", 0.0, L, W.WCA_RC, potential="wca", lattice="sc", K=K, jitter=0.05,
                      extra=extra), 7
