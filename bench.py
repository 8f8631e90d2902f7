#!/usr/bin/env python
"""Benchmark of the cell-list force path (arXiv 1412.3784) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4] [--variant do|ds]

A step is one SLLOD step of the whole hot path (box update and
remap, wrap + cell keys, counting sort, neighborhood + pair kernel, reduction,
kick/drift) on the resident state of BASELINE configs[4] (67,108,864 LJ
particles, planar-elongation KR box, fp32).  Prints ONE JSON line (rank 0).

metric = pair interactions/s (unordered physical pairs |P|/2 per force
evaluation / step time); particle-steps/s is reported beside it.  The timed
region is bracketed by barrier + synchronize, timed with CUDA events on the
library's stream, max over ranks.  Inputs (~100 B/particle, 7 GB) are far
larger than L2 (126 MB), so no L2 flush is needed.

--impl reference times the CPU oracle (oracle/, fp64, the box's host cores)
on the same config and metric, each step a bounded particle sample with the
O(N) cell build amortized per particle.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "force-step throughput: pair interactions/s and particle-steps/s per GPU, % roofline"
UNIT = "pair interactions/s"


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


def dist_setup(backend):
    import torch.distributed as dist

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return rank, lrank, ws


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def relaxed_fluid(w, variant, k, device, iters=200, eta=1e-3, dmax=0.05):
    """BASELINE's fluid input (configs 1-4): positions uniform in fractional
    coordinates, then `iters` capped steepest-descent overlap-removal steps
    q <- q + F min(eta, dmax / |F|), the forces from the library itself (an NC_F64 context, so the
    1e30-scale forces of the first, overlapping configurations stay finite).  Untimed input
    preparation.  Returns fp64 host positions."""
    import torch
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList

    q = torch.from_numpy(W.uniform_positions(w, dtype=np.float64, k=k)).to(device)
    cl = CellList(variant, "f64", rc=w.rc, eps=w.eps, sigma=w.sigma, u_shift=w.ushift, capacity=w.n, max_cells=0,
                  device=torch.device(device).index or 0)
    cl.set_box(w.L)
    F = torch.empty_like(q)
    for _ in range(iters):
        cl.compute_forces(q, F)
        fn = torch.linalg.vector_norm(F, dim=1, keepdim=True).clamp_min(1e-300)
        q.add_(F * torch.clamp(dmax / fn, max=eta))
    fmax = float(torch.linalg.vector_norm(F, dim=1).max())
    cl.close()
    out = q.cpu().numpy()
    del q, F
    torch.cuda.empty_cache()
    return out, fmax


def tier_split(cl, dt):
    """Fraction of the interactions the fp32 far tier evaluates, measured by one extra (untimed)
    SLLOD step with k_pairs' counting instantiation (nc_profile mode 3) after the timed region."""
    cl.profile(3)
    cl.step(dt, 1, want_uw=False)
    st = cl.stats()
    cl.profile(False)
    return st["acc_interactions_fp32"] / max(st["acc_interactions"], 1.0)


def l2_text(n):
    mb = n * 190 / 1e6  # resident bytes per particle in fp32 mode
    if mb > 126:
        return f"inputs (~{mb / 1e3:.1f} GB) >> L2 (126 MB); no flush"
    return f"inputs (~{mb:.0f} MB) fit in L2 (126 MB), no flush: a per-config line, not the bench workload"


def box_text(w):
    return {"none": "equilibrium cube", "le": "Lees-Edwards shear", "kr": "KR planar elongation",
            "gkr": "generalized KR " + str(w.extra.get("flow", ""))}[w.policy] + f", dt={w.dt}"


def pot_text(w):
    return ("WCA" if w.potential == "wca" else "LJ") + f" rc={w.rc:.4f} shifted"


def workload(k: int):
    from paper_1412_3784_b200 import workloads as W

    return W.make(k)


def oracle_sample(w, q32, sample: int, seed: int = 0, prec: str = "f32", variant: str = "do"):
    """The CPU oracle as it stands on a bounded sample of the workload: full O(N)
    cell-list build (the bench's variant), pair loop for `sample` random particles; extrapolated to
    one full force evaluation.  Returns (interactions/s unordered, seconds per
    full evaluation, sample description, threads)."""
    import oracle

    qo = oracle.wrap(q32.astype(np.float64), w.L, prec)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(len(qo), size=sample, replace=False))
    r = oracle.evaluate(oracle.DS if variant == "ds" else oracle.DO, qo, w.L, w.rc, w.eps, w.sigma, w.ushift, idx=idx, want=())
    n = len(qo)
    t_full = r.t_build + r.t_eval * (n / sample)
    inter_full = r.interactions * (n / sample) / 2.0
    return inter_full / t_full, t_full, r, oracle.num_threads()


def run_reference(args):
    """--impl reference: the oracle as it stands, on host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = workload(args.config)
    from paper_1412_3784_b200 import workloads as W

    prec = args.prec or w.prec[0]
    q = W.positions(w, dtype=np.float32 if prec == "f32" else np.float64, k=args.config)
    sample = min(args.ref_sample, w.n)
    vals, times = [], []
    for s in range(args.warmup + args.steps):
        v, tf, r, thr = oracle_sample(w, q, sample, seed=s, prec=prec, variant=args.variant)
        if s >= args.warmup:
            vals.append(v)
            times.append(tf)
    value = len(vals) / sum(1.0 / v for v in vals)  # harmonic mean = total work / total time
    ms = 1e3 * statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded jittered lattice in fractional coordinates, DESIGN.md section 4)",
        "config": {"workload": f"C{args.config}", "n": w.n, "variant": args.variant, "box": box_text(w)},
        "ms_per_step_note": "extrapolated: each step is the O(N) cell build plus a bounded particle sample, "
                            "scaled to one force evaluation of all particles",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"per step: full O(N) {args.variant.upper()} cell build + pair loop of {sample} random particles, "
                                   f"extrapolated to one force evaluation of all {w.n}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_slab(args):
    """N > 1: slab decomposition of C4 over the ranks (strong scaling), NCCL P2P halo
    exchange and migration (paper_1412_3784_b200/slab.py)."""
    import torch
    import torch.distributed as dist

    rank, lrank, ws = dist_setup("nccl")
    torch.cuda.set_device(lrank)
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList
    from paper_1412_3784_b200.slab import SlabRankDev, SlabSystem, own_particles

    # --weak: 8,388,608 particles per GPU in a box elongated along v3; else C<k> split
    w = W.make_weak(ws) if args.weak else workload(args.config)
    kq = args.config if not args.weak else 4
    # the same input as the single-GPU line (BASELINE's relaxed fluid unless --input lattice); every rank
    # relaxes the same seeded system (deterministic) and keeps its own slab
    input_kind = args.input if (args.weak or args.config != 0) else "lattice"
    relax_fmax = None
    if input_kind == "fluid":
        qf, relax_fmax = relaxed_fluid(w, args.variant, kq, f"cuda:{lrank}")
        q = qf.astype(np.float32)
        del qf
    else:
        q = W.positions(w, dtype=np.float32, k=kq, r=0)
    p = W.momenta(w, dtype=np.float32, k=kq, r=0)
    kw = dict(L0=w.L0)
    if w.policy == "kr":
        kw["tstar"] = w.extra["tstar"]
    if w.policy == "gkr":
        kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
    maxc = 0
    # a small context with the full box splits the particles by layer (chunks of 2^20): no full-size
    # context per rank
    full = CellList(args.variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=1 << 20, max_cells=2 * w.n + 4096,
                    device=lrank)
    full.set_flow(w.A, w.policy, w.t0, **kw)
    idx = own_particles(full, torch.from_numpy(q).to(f"cuda:{lrank}"), rank, ws)
    from paper_1412_3784_b200 import nemdcell as ncm
    l3 = int(ncm.nc_slab_layers(full.ctx, 0, 1)[2])
    full.close()
    torch.cuda.empty_cache()
    stream = torch.cuda.Stream(lrank)
    cap = int(1.15 * w.n / ws) + 4 * w.n // l3 + 65536
    # the host-synchronization-free step (SlabRankDev): fixed-capacity halo messages of 1.5 layers,
    # migration messages of 1/8 layer (a step moves ~0.1% of a boundary layer)
    layer = w.n // l3
    if os.environ.get("NC_SLAB_HOSTCOUNTS") == "1":  # A/B: the round-1 step with host-read counts
        from paper_1412_3784_b200.slab import SlabRank
        sr = SlabRank(rank, ws, variant=args.variant, prec="f32", rc=w.rc, u_shift=w.ushift, mass=w.mass,
                      capacity=cap, max_cells=maxc, device=lrank, stream=stream.cuda_stream)
    else:
        sr = SlabRankDev(rank, ws, variant=args.variant, prec="f32", rc=w.rc, u_shift=w.ushift, mass=w.mass,
                         capacity=cap, hcap=int(1.5 * layer) + 4096, mcap=layer // 8 + 4096, max_cells=maxc,
                         device=lrank, stream=stream.cuda_stream)
    sr.set_flow(w.A, w.policy, w.t0, **kw)
    sr.load(q[idx], p[idx], idx.astype(np.int32))
    del q, p
    from paper_1412_3784_b200.slab import LoopbackTransport, NcclTransport

    # N > 1: the library's own NCCL data plane (whole fixed-capacity messages, nc_sd_exchange_start /
    # nc_slab_allgather); torch only broadcasts the unique id.  No host synchronization inside a step.
    if ws == 1:
        tr = LoopbackTransport()
    elif args.transport == "ipc":  # the packing kernels write the neighbours' receive buffers (peer memory)
        from paper_1412_3784_b200.slab import IpcTransport
        tr = IpcTransport(sr, rank, ws)
    else:
        tr = NcclTransport(sr, rank, ws)
    sysm = SlabSystem([sr], tr)
    with torch.cuda.stream(stream):
        sysm.forces(False)
        for _ in range(args.warmup):
            sysm.step(w.dt, False)
    torch.cuda.synchronize()
    sampler = ClockSampler(lrank)
    sr.cl.profile(5)  # pair-kernel events only inside the timed region (breakdown: untimed pass below)
    l0 = sr.cl.launches()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            sysm.step(w.dt, False)
        ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    if hasattr(sr, "status"):
        sr.status()  # after the timed region: raises if a message or the own capacity overflowed
    ms = ev0.elapsed_time(ev1)
    launches = sr.cl.launches() - l0
    prof = sr.cl.profile_read()
    st = sr.cl.stats()
    nprof = max(1, min(args.steps, 5))
    sr.cl.profile(True)
    with torch.cuda.stream(stream):
        for _ in range(nprof):
            sysm.step(w.dt, False)
    prof_all = sr.cl.profile_read()
    sr.cl.profile(False)
    t = torch.tensor([ms, st["acc_interactions"], st["acc_candidates"], float(launches)], dtype=torch.float64,
                     device=f"cuda:{lrank}")
    tmax = t.clone()
    if ws > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t)
    ms_max = float(tmax[0])
    inter = float(t[1])
    value = inter / 2.0 / (ms_max * 1e-3)

    # roofline of rank 0's pair kernel (its own cells: flops from its stats, time from its events)
    evals = max(st["acc_evals"], 1)
    pairs_ms, pairs_n = prof["pairs"]
    cand0, inter0 = st["acc_candidates"] / evals, st["acc_interactions"] / evals
    sr.cl.profile(3)  # one untimed step with k_pairs' tier counting (all ranks step together)
    with torch.cuda.stream(stream):
        sysm.step(w.dt, False)
    stream.synchronize()
    st3 = sr.cl.stats()
    sr.cl.profile(False)
    split = st3["acc_interactions_fp32"] / max(st3["acc_interactions"], 1.0)
    nsm = torch.cuda.get_device_properties(lrank).multi_processor_count
    fmax = (load_peaks().get("sm_max_mhz") or 1965.0) * 1e6
    p32 = nsm * 128 * 2 * fmax
    p64 = p32 / 2.0
    flops0 = 9.0 * cand0 + 30.0 * inter0
    t_bound = (9.0 * cand0 + 30.0 * inter0 * split) / p32 + 30.0 * inter0 * (1.0 - split) / p64
    # a slab evaluation launches k_pairs three times (interior layers, then the two boundary layers
    # after the halo arrives): time per EVALUATION
    pairs_eval_ms = pairs_ms / evals
    achieved = flops0 / (pairs_eval_ms * 1e-3) / 1e12
    roof = {"bound": "alu", "achieved": achieved, "peak": p32 / 1e12, "unit": "TFLOP/s",
            "frac": achieved / (p32 / 1e12), "traffic": None, "kernel": "k_pairs (rank 0)",
            "kernel_ms": pairs_eval_ms, "launches_per_eval": pairs_n / evals,
            "peak_note": f"FP32 {p32/1e12:.1f} TFLOP/s ({nsm} SMs x 128 x 2 x {fmax/1e6:.0f} MHz)",
            "peak_blend": flops0 / t_bound / 1e12, "frac_blend": achieved / (flops0 / t_bound / 1e12),
            "peak_blend_note": f"FP32/FP64 blend; {split:.1%} of rank 0's interactions in the fp32 tier"}

    # end to end through the slab API, pipelined like nc_compute_forces_async: every evaluation each
    # rank copies its own positions from pinned host memory (copy stream, double-buffered, issued
    # one evaluation ahead), runs the halo exchange + forces, and copies F back (second copy stream)
    n_own = sr.n
    qh = torch.empty((n_own, 3), dtype=torch.float32, pin_memory=True)
    Fh = torch.empty((n_own, 3), dtype=torch.float32, pin_memory=True)
    qh.copy_(sr.q[:n_own])
    qbuf = [torch.empty((n_own, 3), dtype=torch.float32, device=f"cuda:{lrank}") for _ in range(2)]
    Fbuf = [torch.empty((n_own, 3), dtype=torch.float32, device=f"cuda:{lrank}") for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(lrank), torch.cuda.Stream(lrank)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]  # qbuf[b] consumed / Fbuf[b] copied out
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()

    def copy_in(b):
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_used[b])
            qbuf[b].copy_(qh, non_blocking=True)
            ev_in[b].record(s_in)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        copy_in(0)
        for k in range(args.steps):
            b = k % 2
            if k + 1 < args.steps:
                copy_in(1 - b)  # next evaluation's input travels during this one
            stream.wait_event(ev_in[b])
            sr.q[:n_own].copy_(qbuf[b], non_blocking=True)
            sysm.forces(False)
            Fbuf[b].copy_(sr.F[:n_own], non_blocking=True)
            ev_out[b].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_out[b])
                Fh.copy_(Fbuf[b], non_blocking=True)
                ev_used[b].record(s_out)
        stream.wait_stream(s_out)
        e1.record(stream)
    e1.synchronize()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{lrank}")
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": inter / 2.0 / (float(te[0]) * 1e-3),  # as many evaluations as the timed steps
           "unit": UNIT, "h2d_bytes_per_step": int(12 * w.n), "d2h_bytes_per_step": int(12 * w.n),
           "call": "slab forces from pinned host q to pinned host F on every rank, copies on two copy streams "
                   "double-buffered and issued one evaluation ahead (as nc_compute_forces_async)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f32",
            "data": ("synthetic fluid: seeded uniform fractional positions + 200 capped steepest-descent overlap-"
                     f"removal steps through the library (max |F| after: {relax_fmax:.3g}), Gaussian momenta T=1"
                     if input_kind == "fluid" else
                     "synthetic (seeded jittered lattice in fractional coordinates, DESIGN.md section 4)"),
            "config": {"workload": w.name if args.weak else f"C{args.config}", "n_total": w.n,
                       "n_per_gpu": w.n // ws, "variant": args.variant, "input": input_kind,
                       "box": box_text(w), "potential": pot_text(w),
                       "precision": "fp32 storage + fp32 filter, fp32/fp64 two-tier interactions",
                       "l2": "inputs >> L2; no flush", "parallelism": f"slabs x{ws} (cell layers along lambda_3), "
                       + ("peer-memory halo + migration written by the packing kernels (CUDA IPC)"
                          if args.transport == "ipc" and ws > 1 else "NCCL P2P halo + migration inside libnemdcell")
                       + ", host-synchronization-free step (fixed-capacity messages, nc_sd_*)"},
            "particle_steps_per_s": w.n * args.steps / (ms_max * 1e-3),
            "kernel_ms_per_step_rank0": {k: v[0] / nprof for k, v in prof_all.items() if v[1]},
            "roofline": roof, "cpu_baseline": None, "e2e": e2e, "gpu_launches": int(t[3]), "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    sr.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch

    rank, lrank, ws = dist_setup("nccl")
    torch.cuda.set_device(lrank)
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList

    w = workload(args.config)
    peaks = load_peaks()
    prec = args.prec or w.prec[0]          # the config's precision (BASELINE: C0 fp64, C1-C4 fp32)
    npdt = np.float32 if prec == "f32" else np.float64
    if args.t0 is not None and w.policy == "kr":  # a point of the KR period (fraction of t*)
        w.t0 = float(args.t0) * w.extra["tstar"]
        w.L = W.box_at(w.L0, w.A, w.policy, w.t0, w.extra)
    # the same seeded workload per rank (independent replicas; slab decomposition is the next row)
    input_kind = args.input if args.config != 0 else "lattice"  # C0 is an FCC crystal by BASELINE's spec
    relax_fmax = None
    if input_kind == "fluid":
        qf, relax_fmax = relaxed_fluid(w, args.variant, args.config, f"cuda:{lrank}")
        q = qf.astype(npdt)
        del qf
    else:
        q = W.positions(w, dtype=npdt, k=args.config, r=0)
    p = W.momenta(w, dtype=npdt, k=args.config, r=0)
    stream = torch.cuda.Stream(lrank)
    cl = CellList(args.variant, prec, rc=w.rc, eps=w.eps, sigma=w.sigma, u_shift=w.ushift, mass=w.mass,
                  capacity=w.n, max_cells=0, device=lrank, stream=stream.cuda_stream)
    if args.pair_kernel != "auto":
        cl.pair_kernel(args.pair_kernel)
    kw = dict(L0=w.L0)
    if w.policy == "kr":
        kw["tstar"] = w.extra["tstar"]
    if w.policy == "gkr":
        kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
    cl.set_flow(w.A, w.policy, w.t0, **kw)
    qd = torch.from_numpy(q).to(f"cuda:{lrank}")
    pd = torch.from_numpy(p).to(f"cuda:{lrank}")
    cl.set_state(qd, pd)
    del qd, pd
    dt = w.dt
    # --steps-per-call: SLLOD steps per nc_step_sllod call (the API takes a step count); 1 = one call
    # per step (default), 0 = all K timed steps in one call (measured equal on C0-C4: the host
    # overhead per call is hidden behind the queued launches)
    spc = args.steps_per_call if args.steps_per_call > 0 else max(args.steps, 1)

    def run_steps(k):
        while k > 0:
            m = min(k, spc)
            cl.step(dt, m, want_uw=False)
            k -= m

    run_steps(args.warmup)
    torch.cuda.synchronize()

    import torch.distributed as dist

    def barrier():
        if ws > 1:
            dist.barrier()

    sampler = ClockSampler(lrank)
    # inside the timed region only the pair kernel carries events (nc_profile bit 4: two per step, for the
    # roofline's live per-launch time); the per-kernel breakdown comes from an untimed pass afterwards
    cl.profile(5)
    l0 = cl.launches()
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # one event per call boundary as well (median and min per step beside the mean)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev0.record(stream)
    if spc == 1:
        evs[0].record(stream)
        for k in range(args.steps):
            cl.step(dt, 1, want_uw=False)
            evs[k + 1].record(stream)
    else:
        run_steps(args.steps)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    per_step = sorted(evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)) if spc == 1 else []
    barrier()
    clocks = sampler.stop()
    ms_total = ev0.elapsed_time(ev1)
    launches = cl.launches() - l0
    prof = cl.profile_read()
    cl.profile(False)
    st = cl.stats()
    # the per-kernel breakdown: a few untimed steps with events around every launch
    nprof = max(1, min(args.steps, 5))
    cl.profile(True)
    if spc == 1:
        for _ in range(nprof):
            cl.step(dt, 1, want_uw=False)
    else:
        cl.step(dt, nprof, want_uw=False)
    prof_all = cl.profile_read()
    cl.profile(False)
    if ws > 1:
        t = torch.tensor([ms_total], device=f"cuda:{lrank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        tot = torch.tensor([st["acc_interactions"], st["acc_candidates"]], dtype=torch.float64, device=f"cuda:{lrank}")
        dist.all_reduce(tot)
        acc_inter, acc_cand = float(tot[0]), float(tot[1])
    else:
        acc_inter, acc_cand = st["acc_interactions"], st["acc_candidates"]
    evals = st["acc_evals"]
    secs = ms_total * 1e-3
    value = (acc_inter / 2.0) / secs
    psteps = w.n * ws * args.steps / secs

    # roofline of the dominant kernel (pair kernel), from live per-launch event times
    pairs_ms, pairs_n = prof["pairs"]
    pairs_ms_avg = pairs_ms / max(pairs_n, 1)
    cand = st["acc_candidates"] / max(evals, 1)
    inter = st["acc_interactions"] / max(evals, 1)
    inter32 = inter * tier_split(cl, dt) if prec == "f32" else 0.0  # evaluated by the fp32 far tier
    inter64 = inter - inter32                                        # by the fp64 close tier
    nsm = torch.cuda.get_device_properties(lrank).multi_processor_count
    fmax = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    p32 = nsm * 128 * 2 * fmax                      # FP32 FMA lanes x 2 flops x clock
    p64 = p32 / 2.0                                 # B200 FP64 = 1/2 FP32
    flops = 9.0 * cand + 30.0 * inter               # SURVEY 8(d3) work model (algorithmic)
    if prec == "f32":
        # each flop at the peak of the precision it is computed in: filter and far tier
        # fp32, close tier fp64 (the measured split of this run)
        t_bound = (9.0 * cand + 30.0 * inter32) / p32 + 30.0 * inter64 / p64
        peak_note = (f"blend of FP32 {p32/1e12:.1f} and FP64 {p64/1e12:.1f} TFLOP/s at {fmax/1e6:.0f} MHz x {nsm} SMs "
                     f"for 9 flop/candidate (fp32) + 30 flop/interaction: {inter32 / max(inter, 1e-30):.1%} of the "
                     f"interactions in the fp32 far tier, the rest in fp64")
    else:
        t_bound = flops / p64                           # NC_F64: every flop in fp64
        peak_note = f"FP64 {p64/1e12:.1f} TFLOP/s at {fmax/1e6:.0f} MHz x {nsm} SMs (NC_F64: all work in fp64)"
    achieved = flops / (pairs_ms_avg * 1e-3) / 1e12
    peak_blend = flops / t_bound / 1e12
    peak = (p32 if prec == "f32" else p64) / 1e12  # the FP32 pair-flop roofline (BASELINE), FP64 for NC_F64
    # the bound that applies: max(T_ALU, T_HBM) with the compulsory force-step bytes
    # (read q, write F, one cell-sorted copy written and read, key + gid: 56 B fp32 / 104 B fp64)
    bytes_p = 56.0 if prec == "f32" else 104.0
    hbm = (peaks.get("hbm_gbs") or 6456.5) * 1e9
    t_alu, t_hbm = flops / (peak * 1e12), bytes_p * w.n / hbm
    roof_bound = "alu" if t_alu >= t_hbm else "hbm"
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(f"C{args.config}-{args.variant}", {}).get("pairs_dram_bytes")
        except Exception:
            traffic = None
    kernel_ms = {k: v[0] / nprof for k, v in prof_all.items() if v[1]}

    # e2e: the same metric through the C-ABI with HOST (pinned) buffers, copies inside the timed region
    e2e = None
    if rank == 0 or True:
        qh = torch.from_numpy(q).pin_memory()  # host positions in the run's precision
        Fh = torch.empty_like(qh).pin_memory()
        cl.set_box(cl_box(cl))
        cl.compute_forces(qh, Fh)  # warm-up
        torch.cuda.synchronize()
        # pipelined host-buffer API: each call copies q in and F out on the library's copy streams,
        # overlapping the neighbouring calls' evaluations; the last call's U, W at the sync
        reps = max(3, args.steps)
        cl.compute_forces_async(qh, Fh)  # warm-up of the async buffers
        cl.compute_sync()
        t0 = time.perf_counter()
        for _ in range(reps):
            cl.compute_forces_async(qh, Fh)
        Ue, _ = cl.compute_sync()
        t1 = time.perf_counter()
        se = cl.stats()
        e2e = {"value": (se["interactions"] / 2.0) / ((t1 - t0) / reps), "unit": UNIT,
               "h2d_bytes_per_step": int(q.nbytes), "d2h_bytes_per_step": int(Fh.numel() * Fh.element_size()),
               "calls": reps,
               "call": f"{reps} x nc_compute_forces_async(pinned host q -> pinned host F) + nc_compute_sync (U, W "
                       f"of the last); wall clock over the calls, copies inside"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        v, tf, r, thr = oracle_sample(w, q, min(args.ref_sample, w.n), prec=prec, variant=args.variant)
        cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"full O(N) {args.variant.upper()} cell build + pair loop of {args.ref_sample} random particles of C{args.config}, "
                         f"extrapolated to one force evaluation ({tf:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            # bench --gpus N > 1 splits C4 over the ranks (strong scaling, run_slab); N = 1 is its first point
            "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": prec,
            "data": ("synthetic fluid: seeded uniform fractional positions + 200 capped steepest-descent overlap-"
                     f"removal steps through the library (max |F| after: {relax_fmax:.3g}), Gaussian momenta T=1"
                     if input_kind == "fluid" else
                     "synthetic (seeded jittered lattice in fractional coordinates, DESIGN.md section 4)"),
            "config": {"workload": f"C{args.config}", "n_per_gpu": w.n, "variant": args.variant, "input": input_kind,
                       "t0": w.t0, "t0_over_period": (w.t0 / w.extra["tstar"] if w.policy == "kr" else None),
                       "box": box_text(w), "potential": pot_text(w),
                       "precision": ("fp32 storage + fp32 filter, fp32/fp64 two-tier interactions" if prec == "f32"
                                     else "fp64 throughout"),
                       "l2": l2_text(w.n), "parallelism": f"replicas x{ws}", "steps_per_call": spc},
            "particle_steps_per_s": psteps,
            "ms_per_step_median": per_step[len(per_step) // 2] if per_step else None,
            "ms_per_step_min": per_step[0] if per_step else None,
            "interactions_per_particle": inter / w.n, "candidates_per_particle": cand / w.n,
            "roofline": ({"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                          "frac": achieved / peak} if roof_bound == "alu" else
                         {"bound": "hbm", "achieved": bytes_p * w.n / (pairs_ms_avg * 1e-3) / 1e9,
                          "peak": hbm / 1e9, "unit": "GB/s", "frac": t_hbm / (pairs_ms_avg * 1e-3)}) | {
                         "traffic": traffic, "kernel": "k_pairs",
                         "kernel_ms": pairs_ms_avg, "t_alu_ms": t_alu * 1e3, "t_hbm_ms": t_hbm * 1e3,
                         "peak_note": (f"FP32 {p32/1e12:.1f} TFLOP/s = {nsm} SMs x 128 x 2 x {fmax/1e6:.0f} MHz"
                                       if prec == "f32" else peak_note) + "; algorithmic flops 9/candidate + "
                                       "30/interaction (SURVEY 8(d3)); bytes 56 B/particle (fp32) / 104 (fp64)",
                         "frac_alu": achieved / peak, "peak_blend": peak_blend, "frac_blend": achieved / peak_blend,
                         "peak_blend_note": peak_note, "pair_kernel": cl.pair_kernel_used()},
            "kernel_ms_per_step": kernel_ms,
            "kernel_ms_note": (f"per-kernel breakdown from {nprof} untimed steps with events around every launch; "
                               "the timed region carries events around the pair kernel only (roofline)"),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    cl.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def cl_box(cl):
    n, L, t, _ = cl.get_state()
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--variant", default="do", choices=["do", "ds"])
    ap.add_argument("--prec", default=None, choices=["f32", "f64"], help="default: the config's precision")
    ap.add_argument("--ref-sample", type=int, default=100000)  # ~20 s of oracle work on the C4 sample
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--steps-per-call", type=int, default=1,
                    help="SLLOD steps per nc_step_sllod call (0 = all timed steps in one call; measured the same)")
    ap.add_argument("--slab", action="store_true", help="use the slab (multi-GPU) path even on one GPU")
    ap.add_argument("--input", default="fluid", choices=["fluid", "lattice"],
                    help="fluid: BASELINE's relaxed uniform positions (default); lattice: the jittered crystal")
    ap.add_argument("--t0", type=float, default=None, help="KR configs: start at t0 = this fraction of t*")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1 data plane: NCCL send/recv of whole messages (default) or peer-memory stores from "
                         "the packing kernels (CUDA IPC, NVLink)")
    ap.add_argument("--pair-kernel", default="auto", choices=["auto", "cell", "segment", "sparse", "rows"],
                    help="force one K3 pair kernel (A/B runs; default: the library's choice)")
    ap.add_argument("--weak", action="store_true",
                    help="slab path, weak scaling: 8,388,608 particles per GPU (box elongated along v3)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.slab or args.weak:
        return run_slab(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
