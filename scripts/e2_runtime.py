"""NEXT item f2: the paper's only runtime experiment: 1728
WCA particles, 10,000 steps, uniaxial flow, DO time / DS time (paper: 71.7% on an
unspecified single-core machine; its volume model predicted ~56%).  Here: the same
system on one B200 through nc_step_sllod (both variants), and the CPU oracle's
force evaluation on ONE core (OMP_NUM_THREADS=1) for the DO/DS ratio of the
pair search itself.  Writes profiles/e2_runtime.json."""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList

    K = 12                                   # 12^3 = 1728 particles, SC lattice at rho = 0.8442
    n = K ** 3
    a = (n / W.RHO) ** (1.0 / 3.0)           # 12.7 sigma -> ~11 WCA cells per direction ("about 10")
    M1, M2, L0, om1, om2 = W.gkr_params(a)
    adiag = np.array([2.0, -1.0, -1.0])
    eps = 0.025
    A = np.diag(eps * adiag)                  # diag(0.05, -0.025, -0.025)
    beta = np.linalg.lstsq(np.stack([om1, om2], axis=1), adiag, rcond=None)[0]
    extra = {"beta": beta, "eps": eps, "om1": om1, "om2": om2}
    t0 = 0.0
    L = W.box_at(L0, A, "gkr", t0, extra)
    w = W.Workload("E2", n, L0, A, "gkr", t0, L, W.WCA_RC, potential="wca", lattice="sc", K=K, jitter=0.05,
                   extra=extra)
    q = W.positions(w, dtype=np.float32, k=7)
    p = W.momenta(w, dtype=np.float32, k=7)
    steps, dt = 10000, 0.002
    out = {"n": n, "a": a, "steps": steps, "dt": dt, "paper_P747": {"do_over_ds": 0.717, "predicted": 0.56}}
    snaps = []  # (q, L) every 100 steps of the DO run: the boxes the single-core oracle is timed on
    for v in ("ds", "do"):
        cl = CellList(v, "f32", rc=W.WCA_RC, u_shift=w.ushift, capacity=n, max_cells=1 << 16)
        cl.set_flow(A, "gkr", t0, L0=L0, om1=om1, om2=om2, beta=beta, eps=eps)
        cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
        cl.step(dt, 200, want_uw=False)
        torch.cuda.synchronize()
        # the run, no instrumentation inside (one nc_step_sllod call; U, W read once at the end)
        t1 = time.perf_counter()
        U, _ = cl.step(dt, steps)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        st = cl.stats()  # candidates over the timed run (the second run below continues the trajectory)
        # the same number of steps again with events around the pair kernel (its share; the two events
        # break the programmatic-dependent-launch overlap at its boundaries, so this run is slower)
        cl.profile(5)
        t3 = time.perf_counter()
        cl.step(dt, steps)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        if v == "do":  # the same trajectory again, sampled every 100 steps (not timed)
            cl.set_flow(A, "gkr", t0, L0=L0, om1=om1, om2=om2, beta=beta, eps=eps)
            cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
            cl.step(dt, 200, want_uw=False)
            qh = torch.empty((n, 3), dtype=torch.float32, device="cuda")
            for _ in range(steps // 100):
                cl.step(dt, 100, want_uw=False)
                _, Ls, _, _ = cl.get_state(qh)
                snaps.append((qh.cpu().numpy().astype(np.float64), Ls.copy()))
        prof = cl.profile_read()
        out["gpu_" + v] = {"s_total": t2 - t1, "us_per_step": 1e6 * (t2 - t1) / steps,
                           "us_per_step_with_pair_events": 1e6 * (t4 - t3) / steps,
                           "pairs_kernel_us_per_step": 1e3 * prof["pairs"][0] / max(prof["pairs"][1], 1),
                           "candidates_per_particle": st["acc_candidates"] / max(st["acc_evals"], 1) / n,
                           "U_end": U}
        cl.close()
    out["gpu_do_over_ds_step"] = out["gpu_do"]["us_per_step"] / out["gpu_ds"]["us_per_step"]
    out["gpu_do_over_ds_pairs_kernel"] = out["gpu_do"]["pairs_kernel_us_per_step"] / out["gpu_ds"]["pairs_kernel_us_per_step"]
    out["candidates_do_over_ds"] = out["gpu_do"]["candidates_per_particle"] / out["gpu_ds"]["candidates_per_particle"]
    # single-core oracle force evaluations (cell build + pair loop, OMP_NUM_THREADS=1 set by the caller)
    # on the boxes and states of the run: every 100th step of the 10,000 (P:747 times the whole run)
    try:
        import oracle

        times = {"ds": 0.0, "do": 0.0}
        cand = {"ds": 0.0, "do": 0.0}
        for qs, Ls in snaps:
            qo = oracle.wrap(qs, Ls, "f32")
            for v, m in (("ds", oracle.DS), ("do", oracle.DO)):
                best = None
                for _ in range(3):  # best of three per box (timer noise on ~ms evaluations)
                    r = oracle.evaluate(m, qo, Ls, W.WCA_RC, ushift=w.ushift, want=("F",))
                    tt = r.t_build + r.t_eval
                    best = tt if best is None else min(best, tt)
                times[v] += best
                cand[v] += r.candidates
        out["oracle_threads"] = oracle.num_threads()
        out["oracle_boxes"] = len(snaps)
        out["oracle_seconds"] = times
        out["oracle_do_over_ds_run"] = times["do"] / times["ds"]
        out["oracle_do_over_ds_candidates_run"] = cand["do"] / cand["ds"]
    except Exception as e:  # noqa: BLE001
        out["oracle_error"] = str(e)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "e2_runtime.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
