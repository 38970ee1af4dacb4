#!/usr/bin/env python
"""bench.py — callback + condensed-KKT-assembly throughput on B200.

One *step* = one IPM iteration's hot-path unit of work over
the whole (per-rank) horizon:
    eval_f, eval_grad, eval_g, eval_jac, eval_hess(x, w = -y, 1)
    + set_jacobian(J) + assemble(H, Sigma_x, Sigma_s, dw, dc)
Workload at N=1: BASELINE.json configs[4], the synthetic 30k-bus network x 96
periods (15.26M variables).  Under torchrun each rank owns 96 consecutive
periods of a 96*N-period horizon (weak scaling; period sharding).

`value` is nnz/s: (J + H + M nonzeros produced per step, summed over ranks)
divided by the max-over-ranks device time per step.  `e2e` is the same metric
through the public C-ABI with HOST buffers (every step copies its inputs H2D
from pinned memory and its outputs D2H), i.e. the reference's std::span
drop-in.  `--impl reference` times the reference's own CPU implementation
(oracle/_ref) on the host cores instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "callback+KKT-assembly nnz/s (J+H+M per IPM iteration)"
UNIT = "nnz/s"
PERIODS_PER_RANK = 96
CONFIG = "synthetic30k"
# BASELINE.json `configs` index of each workload (configs[0], case118 x 1, is the CPU parity case)
CONFIG_INDEX = {"case118": 0, "case1354pegase": 1, "case9241pegase": 2, "case13659pegase": 3,
                "synthetic30k": 4}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def inputs(nlp_bounds, m, n_free, seed_shift=0):
    from helpers import interior_point, row_weights, sigmas
    xl, xu, xs = nlp_bounds
    x = interior_point(xl, xu, xs, 1234 + seed_shift)
    w = row_weights(m, 7 + seed_shift)
    sx, ss = sigmas(n_free, m, 11 + seed_shift)
    return x, w, sx, ss


class Clocks:
    """SM clocks and throttle reasons sampled every ~2 ms during the timed region
    (NVML; B200_PROFILING.md clocks line)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index: int):
        import threading
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[index].isdigit() else index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                clk = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                names = [n for n, a in self.REASONS.items() if r & getattr(nv, a, 0)]
                self.samples.append((time.perf_counter(), clk, names))
            except Exception:
                pass
            time.sleep(0.002)

    def mark(self):
        return time.perf_counter()

    def close(self):
        if self.nv is not None and not self._stop.is_set():
            self._stop.set()
            self.t.join(timeout=5)

    def stop(self, t0, t1):
        """Samples taken inside [t0, t1] (at least the 3 nearest when the timed
        region is shorter than the NVML sampling period).  The sampler keeps running:
        several timed windows can be read; close() ends it."""
        if self.nv is None:
            return None
        samples = list(self.samples)
        if not samples:
            return None
        inside = [x for x in samples if t0 <= x[0] <= t1]
        widened = len(inside) < 3
        if widened:
            mid = 0.5 * (t0 + t1)
            inside = sorted(samples, key=lambda x: abs(x[0] - mid))[:3]
        reasons = sorted({n for x in inside for n in x[2]})
        return {"sm_mhz": float(np.median([x[1] for x in inside])),
                "sm_max_mhz": float(self.max_mhz), "reasons": reasons, "samples": len(inside),
                "window_widened": widened}


# ------------------------------------------------------------------ workload
def shard_of(rank: int, world: int, periods: int, strong: bool):
    """(T_total, first period, periods) of this rank: weak scaling = `periods` per rank of a
    world * periods horizon; strong = a `periods` horizon partitioned over the ranks."""
    if not strong:
        return periods * world, periods * rank, periods
    from paper_2405_14032_b200.shard import partition
    t0, T = partition(periods, world)[rank]
    return periods, t0, T


def build_workload(rank: int, world: int, periods: int, config: str, strong: bool = False):
    from paper_2405_14032_b200.network import config_case
    from paper_2405_14032_b200.opf import load_profile
    raw = config_case(config, seed=1)
    net = raw.network()
    T_total, first, T = shard_of(rank, world, periods, strong)
    scale = load_profile(net.n_load, T_total, seed=1)
    return raw, net, np.ascontiguousarray(scale[first:first + T])


def alg_bytes(s, kkt):
    """SURVEY §8(d) B_alg per unit of work (index/scatter maps excluded)."""
    n, m, J, H = s.n_vars, s.n_cons, s.jac_nnz, s.hess_nnz
    Jl, Hl, nl, M = s.jac_nnz_lifted, s.hess_nnz_lifted, s.n_free, kkt.m_nnz
    return 8 * (2 * n + 2 * m + 1 + J + H) + 8 * (Jl + Hl + nl + m + M)


def stage_bytes(s, kkt, net, periods, fused=False):
    """Algorithmic bytes per call (contract inputs read once + outputs written once)."""
    n, m, J, H = s.n_vars, s.n_cons, s.jac_nnz, s.hess_nnz
    GT = net.n_gen * periods
    if fused:  # A, M from x: x (+ w, sigma) read once, A / M written once
        return {
            "f": 8 * (GT + 1), "grad": 8 * (n + GT), "g": 8 * (n + m), "jac": 8 * (n + J),
            "hess": 8 * (n + m + H),
            "set_jacobian": 8 * (n + kkt.a_nnz),
            "assemble": 8 * (n + 2 * m + s.n_free + kkt.m_nnz),
        }
    return {
        "f": 8 * (GT + 1),
        "grad": 8 * (n + GT),
        "g": 8 * (n + m),
        "jac": 8 * (n + J),
        "hess": 8 * (n + m + H),
        "set_jacobian": 8 * (s.jac_nnz_lifted + kkt.a_nnz),
        "assemble": 8 * (s.hess_nnz_lifted + kkt.a_nnz + s.n_free + m + kkt.m_nnz),
    }


def kernel_bytes(s, kkt, nlp, net, T):
    """Algorithmic bytes per launch of each library kernel: the contract outputs
    it writes once plus the inputs it needs read once (index maps excluded)."""
    N, L, G, D = net.n_bus, net.n_line, net.n_gen, net.n_load
    LTh, GR = s.n_thermal, s.n_ramp_gens
    R = max(T - 1, 0)
    m, annz = s.n_cons, kkt.a_nnz
    # M slots per column block, from the lifted structure
    rowptr, _, colptr, _ = kkt.structure()
    a_flow = int(rowptr[2 * N * T + 2 * L * T] - rowptr[2 * N * T])  # A entries of flow rows
    lens = np.diff(colptr.astype(np.int64))
    f2f = nlp.lifted_structure()["free_to_full"]
    bounds = np.cumsum([0, G * T, G * T, L * T, L * T, N * T, N * T])
    blk = np.searchsorted(bounds, f2f, side="right") - 1  # 0 pg 1 qg 2 p 3 q 4 v 5 th
    deg = np.bincount(np.concatenate([net.line_from, net.line_to]), minlength=N)
    ent = np.where(blk >= 4, (f2f - bounds[np.minimum(blk, 5)]) // T, -1)
    vth = (blk == 4) | (blk == 5)
    m_pq = int(lens[(blk == 2) | (blk == 3)].sum())
    m_g = int(lens[blk <= 1].sum())
    # bus-column kernels by class (as the library forms them): buses of exactly D = 1..6
    # lines without parallel lines -> k_fz_busr<dD>; the others -> k_fz_bus3<le8> (<= 8
    # lines) / k_fz_bus3<rest>.  Per class: its M slots, x(v, th) + Sx(v, th) of its
    # buses, and its share (half per line end) of the line inputs w(flow_p, flow_q),
    # d(flow_p, flow_q, angle)
    lo_ = np.minimum(net.line_from, net.line_to).astype(np.int64)
    hi_ = np.maximum(net.line_from, net.line_to).astype(np.int64)
    key = lo_ * N + hi_
    uk, cnt = np.unique(key, return_counts=True)
    par = np.zeros(N, bool)
    dup = uk[cnt > 1]
    par[(dup // N)] = True
    par[(dup % N)] = True
    # (register classes d1..d7, GN_BUS_REGMAX; every other bus in the one slot-program class)
    simple = (deg >= 1) & (deg <= 7) & ~par
    cls = np.where(simple, deg - 1, 8)
    names = ["k_fz_busr<d1>", "k_fz_busr<d2>", "k_fz_busr<d3>", "k_fz_busr<d4>", "k_fz_busr<d5>",
             "k_fz_busr<d6>", "k_fz_busr<d7>", "k_fz_bus3<le8>", "k_fz_bus3<rest>"]
    m_cls = [int(lens[vth & (cls[np.clip(ent, 0, N - 1)] == k)].sum()) for k in range(9)]
    bus_cls = {nm: m_cls[k] + 4 * int((cls == k).sum()) * T + 2.5 * int(deg[cls == k].sum()) * T
               for k, nm in enumerate(names)}
    # balance rows (bus), flow / angle / thermal rows (line), ramp rows
    cb_g = ((2 * N * T + 2 * L * T + 2 * G * T + 2 * D * T) + (5 * L * T + 2 * N * T + 3 * LTh * T)
            + (GR * R + G * T))
    b = {
        # one launch per callback: its element classes' block ranges (gn_eval.cu); the five in
        # one launch (gn_eval_all, small problems): their sum plus the gradient's zero fill
        "k_eval<ALL>": (G * T + 2 * G * T + cb_g
                        + 16 * L * T + 2 * N * T + 4 * LTh * T + 2 * G * T + 2 * GR * R
                        + 39 * L * T + 2 * N * T + 6 * LTh * T + 4 * G * T + 3 * GR * R
                        + (s.n_vars - G * T)),
        "k_eval<F>": G * T, "k_eval<GRAD>": 2 * G * T,
        "k_eval<G>": cb_g, "k_eval<FG>": cb_g + G * T,
        # line (+ thermal) records, generator and ramp records
        "k_eval<J>": 16 * L * T + 2 * N * T + 4 * LTh * T + 2 * G * T + 2 * GR * R,
        "k_eval<H>": 39 * L * T + 2 * N * T + 6 * LTh * T + 4 * G * T + 3 * GR * R,
        "k_opf_set_jac_fused": annz - 2 * LTh * T + 2 * N * T,
        "k_opf_set_jac_fused<noflow>": annz - a_flow + 2 * LTh * T,
        "k_opf_set_jac_thermal": 4 * LTh * T,
        "k_fz_dvec": 2 * m,
        **bus_cls,
        "k_fz_line": m_pq + 2 * L * T + 2 * N * T + 2 * N * T + 2 * L * T + 2 * LTh * T + 2 * L * T,
        "k_fz_gen": m_g + 2 * G * T + GR * R + 2 * G * T,
        "k_opf_set_jac": 2 * annz, "k_set_jac_generic": 2 * annz,
        "k_opf_assemble": s.hess_nnz_lifted + annz + s.n_free + m + kkt.m_nnz,
        "k_assemble_generic": s.hess_nnz_lifted + annz + s.n_free + m + kkt.m_nnz,
    }
    return {k: 8.0 * v for k, v in b.items()}


def ipm_vector_ops(nlp, kkt, J, grad, g, dsx, dss, flush, stream, peak, reps=5):
    """One IPM iteration's vector work on the device: residuals (with
    J^T y), kkt_error, bound condensation, the condensed solve's rhs and ds/dy around the
    (host, out-of-scope) factor solve, bound-step recovery, fraction to boundary, barrier
    value and slope -- everything an IpmSolver iteration does besides the callbacks, the
    KKT assembly and the LDL^T.  Synthetic interior iterate; L2 flushed before each rep."""
    import torch
    from paper_2405_14032_b200.opf import Ipm
    s = nlp.sizes
    n, m, nj = s.n_free, s.n_cons, s.jac_nnz_lifted
    st = nlp.lifted_structure()
    f2f = st["free_to_full"]
    xl_f, xu_f, xs_f, _, _ = nlp.bounds()
    xl, xu, sl, su = xl_f[f2f], xu_f[f2f], st["s_lower"], st["s_upper"]
    dev = grad.device
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev)  # noqa: E731
    ipm = Ipm(kkt, xl, xu, sl, su)
    rng = np.random.default_rng(3)

    def interior(lo, hi, k):
        base = np.where(np.isfinite(lo), lo, np.where(np.isfinite(hi), hi - 2.0, 0.0))
        width = np.where(np.isfinite(lo) & np.isfinite(hi), hi - lo, 2.0)
        return base + (0.1 + 0.8 * rng.random(k)) * width
    it = [t(interior(xl, xu, n)), t(interior(sl, su, m)), t(rng.uniform(-1, 1, m))]
    it += [t(np.where(np.isfinite(b), rng.uniform(0.01, 2, k), 0.0))
           for b, k in ((xl, n), (xu, n), (sl, m), (su, m))]
    del xl_f, xu_f, xs_f
    jl = torch.empty(nj, dtype=torch.float64, device=dev)
    from paper_2405_14032_b200.opf import _f64
    nlp.lib.gn_lifted_gather_jac(nlp.h, _f64(J), _f64(jl), abi_dev_async())
    e = lambda k: torch.empty(k, dtype=torch.float64, device=dev)  # noqa: E731
    r = [e(k) for k in (n, m, m, n, n, m, m)]
    d = [e(k) for k in (n, m, m, n, n, m, m)]
    sx_, ss_, qx, qs, rhs = e(n), e(m), e(n), e(m), e(n)
    gl = grad[torch.from_numpy(f2f.astype(np.int64)).to(dev)]  # lifted gradient
    kkt.set_jacobian(jl, mem=abi_dev_async())

    def iteration():
        ipm.residuals(it, gl, g, jl, 0.1, r, sync=False)
        ipm.kkt_error(it, r, 0.1, sync=False)
        ipm.bound_condensation(it, r, sx_, ss_, qx, qs, sync=False)
        ipm.solve_rhs(qx, qs, r[2], ss_, 1e-4, 0.0, rhs, sync=False)
        d[0].copy_(rhs)  # stands in for the host LDL^T solve (out of scope)
        ipm.solve_finish(d[0], qs, r[2], ss_, 1e-4, 0.0, d[1], d[2], sync=False)
        ipm.recover_bound_steps(it, r, d, sync=False)
        ipm.fraction_to_boundary(it, d, 0.99, sync=False)
        ipm.barrier_value(1.0, it[0], it[1], 0.1, sync=False)
        ipm.barrier_slope(gl, it, d, 0.1, sync=False)

    with torch.cuda.stream(stream):
        iteration()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for a_, b_ in evs:
        with torch.cuda.stream(stream):
            flush.zero_()
            a_.record(stream)
            iteration()
            b_.record(stream)
    torch.cuda.synchronize()
    ms = float(np.median([a_.elapsed_time(b_) for a_, b_ in evs]))
    # per-kernel event times (library KTimer), L2 flushed before each iteration
    from paper_2405_14032_b200 import abi
    L = abi.lib()
    L.gn_profile_reset()
    L.gn_profile_enable(1)
    for _ in range(3):
        with torch.cuda.stream(stream):
            flush.zero_()
            iteration()
    torch.cuda.synchronize()
    L.gn_profile_enable(0)
    kern = {}
    for i in range(L.gn_profile_count()):
        kms, kn = C.c_double(), C.c_int64()
        name = L.gn_profile_get(i, C.byref(kms), C.byref(kn)).decode()
        if name.startswith("k_ipm"):
            kern[name] = round(kms.value / 3, 5)  # ms per iteration
    L.gn_profile_reset()
    annz = kkt.a_nnz
    vec = {  # algorithmic reads + writes per op, in doubles (index maps excluded)
        "residuals": nj + (4 * n + 5 * m) + (n + m) + 2 * (n + m) + (3 * n + 4 * m),
        "kkt_error": (3 * n + 4 * m) + (n + 2 * m) + 2 * (n + m),
        "bound_condensation": (3 * n + 3 * m) + (3 * n + 3 * m) + 2 * (n + m) + 2 * (n + m),
        "solve_rhs": 3 * m + n + annz + n + 2 * m,
        "rhs_copy": 2 * n,
        "solve_finish": annz + n + 3 * m + 2 * m,
        "recover_bound_steps": 10 * (n + m),  # w, d, z, pz, bounds in; dz out
        "fraction_to_boundary": 8 * (n + m),  # w, d, z, dz, bounds
        "barrier_value": (n + m) + 2 * (n + m),
        "barrier_slope": n + 2 * (n + m) + 2 * (n + m),
    }
    alg = 8.0 * sum(vec.values())
    ipm.close()
    return {"ms": ms, "alg_bytes": alg, "gbs": alg / (ms * 1e-3) / 1e9,
            "frac": alg / (ms * 1e-3) / 1e9 / peak, "n": n, "m": m,
            "ops": list(vec.keys()),
            "kernels_ms": dict(sorted(kern.items(), key=lambda kv: -kv[1]))}


def abi_dev_async():
    from paper_2405_14032_b200.abi import GN_MEM_DEVICE_ASYNC
    return GN_MEM_DEVICE_ASYNC


def profile_kernels(L, step, steps, stream, flush):
    """Per-kernel CUDA-event times (library KTimer, events on each kernel's launch
    stream) over `steps` extra steps run serially on one stream, L2 flushed
    between steps as in the timed region."""
    import torch
    L.gn_profile_reset()
    L.gn_profile_enable(1)
    for _ in range(steps):  # (the caller runs this with the KKT grid uncapped)
        with torch.cuda.stream(stream):
            flush.zero_()
        step(serial=True)
    torch.cuda.synchronize()
    L.gn_profile_enable(0)
    out = {}
    for i in range(L.gn_profile_count()):
        ms, n = C.c_double(), C.c_int64()
        name = L.gn_profile_get(i, C.byref(ms), C.byref(n)).decode()
        out[name] = (ms.value / max(n.value, 1), n.value)
    L.gn_profile_reset()
    return out


def run_ours(args, rank, world, local_rank, dist):
    import torch
    from paper_2405_14032_b200 import abi
    from paper_2405_14032_b200.abi import GN_IN_FULL, GN_MEM_DEVICE_ASYNC, GN_MEM_HOST
    from paper_2405_14032_b200.opf import CondensedKkt, OpfNlp

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    raw, net, scale = build_workload(rank, world, args.periods, args.config, args.strong)
    T_total, first, T_rank = shard_of(rank, world, args.periods, args.strong)
    t0 = time.time()
    # period shard [first, first + T_rank) of the T_total horizon (world == 1: the whole horizon)
    nlp = OpfNlp(net, T_rank, scale, device=local_rank, shard=(T_total, first))
    stream = torch.cuda.Stream(device=dev, priority=int(os.environ.get("GN_CB_PRIORITY", "0")))
    nlp.set_stream(stream.cuda_stream)
    nlp.lift(1e-4)
    kkt = CondensedKkt(nlp=nlp)
    # with two streams the KKT kernels launch at most 2 CTAs per SM (grid-stride), leaving
    # room for the callback stream's bandwidth-bound kernels beside them (swept: 1, 2, 3, 4,
    # 8 and uncapped, per kernel and uniform; uniform 2 is best)
    grid_cap = args.grid_cap if args.grid_cap >= 0 else (2 if args.streams == 2 else 0)
    kkt.set_grid_cap(grid_cap)
    setup_s = time.time() - t0
    s = nlp.sizes
    xl, xu, xs, _, _ = nlp.bounds()
    x, w, sx, ss = inputs((xl, xu, xs), s.n_cons, s.n_free, seed_shift=rank)
    del xl, xu, xs
    f64 = dict(dtype=torch.float64, device=dev)
    dx = torch.from_numpy(x).to(dev)
    dwt = torch.from_numpy(w).to(dev)
    dsx = torch.from_numpy(sx).to(dev)
    dss = torch.from_numpy(ss).to(dev)
    f = torch.zeros(1, **f64)
    f_global = torch.zeros(1, **f64)
    grad = torch.empty(s.n_vars, **f64)
    g = torch.empty(s.n_cons, **f64)
    J = torch.empty(s.jac_nnz, **f64)
    H = torch.empty(s.hess_nnz, **f64)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    torch.cuda.synchronize()
    dw_reg, dc_reg = 1e-4, 1e-8 * 0.1 ** 0.25  # retry-variant regularization
    A = GN_MEM_DEVICE_ASYNC
    L = abi.lib()
    stages = ["f", "grad", "g", "jac", "hess", "set_jacobian", "assemble"]
    fused = args.pipeline == "fused"
    if fused and not kkt.fused_ready:
        raise SystemExit("fused KKT path unavailable (verification failed)")
    if world > 1 and not fused:
        raise SystemExit("period shards run the fused KKT path")

    # ---- ramp halo: boundary set-points forward/backward, the
    # sigma_s of the boundary ramp rows backward (G doubles each) and the objective
    # partials.  --halo peer (default): gn_halo, the neighbours store straight into this
    # GPU's memory over NVLink / NVSwitch, one kernel per exchange, capturable in the
    # step's CUDA graph; --halo nccl: torch.distributed point-to-point (eager only).
    halo = peer = None
    halo_kind = args.halo
    if world > 1:
        from paper_2405_14032_b200.shard import DeviceHalo, ShardMap
        if halo_kind == "peer":
            # every rank must map every peer region, or none uses them: a rank whose mapping
            # failed would leave its neighbours' exchange kernels waiting for its flags
            ok = 1
            try:
                peer = DeviceHalo(nlp, rank, world)
                peer.connect()
            except Exception as e:  # noqa: BLE001 -- reported, then the NCCL halo instead
                print(f"rank {rank}: peer-memory halo unavailable ({e}); using the NCCL halo",
                      file=sys.stderr)
                ok = 0
            import torch.distributed as tdist
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            tdist.all_reduce(flag, op=tdist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                peer = None
                halo_kind = "nccl"
        if halo_kind != "peer":
            info = nlp.shard_info()
            mp_ = ShardMap(net.n_bus, net.n_line, net.n_gen, s.n_thermal, info["ramp_gens"],
                           T_total, first, T_rank)
            halo = mp_.halo_plan(dev)

    def exchange():
        if peer is not None:
            peer.exchange(dx, dss, DeviceHalo.BOTH, torch.cuda.current_stream().cuda_stream)
        else:
            from paper_2405_14032_b200.shard import exchange_halo
            exchange_halo(halo, dx, dss, rank, stage_cpu=halo_kind == "gloo")

    # Two streams: the callbacks on `stream`, the KKT on `kstream`.  Given x, w
    # and Sigma, f/grad/g/J/H and the fused A/M are independent (the fused KKT
    # recomputes its J/H terms), so a device-resident IPM overlaps them; the
    # contract pipeline must wait for J and H.
    # the KKT stream gets the higher priority: its latency-bound kernels are placed
    # first and the bandwidth-bound callback kernels fill the SMs around them
    prio = int(os.environ.get("GN_KKT_PRIORITY", "-1"))
    kstream = torch.cuda.Stream(device=dev, priority=prio) if args.streams == 2 else stream
    kkt.set_stream(kstream.cuda_stream)
    ev_x = torch.cuda.Event()
    ev_k = torch.cuda.Event()

    # callback issue order on the callback stream (the five calls are independent given x;
    # scripts/gpu_order.sh sweeps it: within 1%).  The stage spans assume the default order.
    cb_order = os.environ.get("GN_CB_ORDER", "f,grad,g,jac,hess").split(",")
    assert sorted(cb_order) == sorted(["f", "grad", "g", "jac", "hess"]), cb_order
    cb_mark = {"f": 1, "g": 2, "jac": 3, "hess": 4}
    # one GPU: the callbacks through gn_eval_all (one launch for small problems, the five
    # launches otherwise -- the library's choice; 1354 x 24 -12%).  Period shards keep the
    # five calls so that the objective exchange runs right behind f.  GN_EVAL_BUNDLE=0: off.
    bundle = world == 1 and os.environ.get("GN_EVAL_BUNDLE", "1") == "1"

    def step(ev=None, serial=False, kkt_wait=None, after_cb=None):
        """One unit; serial=True runs the KKT on the callback stream (per-kernel timing).
        kkt_wait: an extra event the KKT waits for (e2e: its Sigma copy); after_cb: called
        once the callbacks are enqueued (e2e: their device-to-host copies)."""
        ks = stream if serial else kstream
        kkt.set_stream(ks.cuda_stream)  # no-op (no sync) when unchanged: capturable

        def mark(i, st=None):
            if ev is not None:
                ev[i].record(st or stream)
        mark(0)
        if world > 1:
            with torch.cuda.stream(stream):
                exchange()
        ev_x.record(stream)  # x (with its halo) ready
        if fused and ks is not stream:
            ks.wait_event(ev_x)
            if kkt_wait is not None:
                ks.wait_event(kkt_wait)
            mark(6, ks)
            kkt.update_x(dx, dwt, 1.0, dsx, dss, dw_reg, dc_reg, mem=A)  # set_jacobian + assemble
            mark(7, ks)
        if bundle:  # the five callbacks in one launch (gn_eval_all)
            nlp.eval_all(dx, dwt, 1.0, outs=(f, grad, g, J, H), mem=A)
            if world > 1:
                with torch.cuda.stream(stream):
                    if peer is not None:
                        peer.objective(f, f_global, DeviceHalo.BOTH, stream.cuda_stream)
                    else:
                        from paper_2405_14032_b200.shard import global_objective
                        f_global.copy_(global_objective(f, world))
            for i in (1, 2, 3, 4):
                mark(i)
        for name in ([] if bundle else cb_order):
            if name == "hess":
                nlp.eval_device("hess", dx, H, w=dwt, ow=1.0, sync=False)
            else:
                nlp.eval_device(name, dx, {"f": f, "grad": grad, "g": g, "jac": J}[name],
                                sync=False)
            if name == "f" and world > 1:  # the global objective: shard partials in rank
                with torch.cuda.stream(stream):  # order, right behind f (off the tail)
                    if peer is not None:
                        peer.objective(f, f_global, DeviceHalo.BOTH, stream.cuda_stream)
                    else:
                        from paper_2405_14032_b200.shard import global_objective
                        f_global.copy_(global_objective(f, world))
            if name in cb_mark:
                mark(cb_mark[name])
        if after_cb is not None:
            after_cb()
        if fused and ks is not stream:
            ev_k.record(ks)
            stream.wait_event(ev_k)
        elif fused:
            if kkt_wait is not None:
                stream.wait_event(kkt_wait)
            mark(6)
            kkt.update_x(dx, dwt, 1.0, dsx, dss, dw_reg, dc_reg, mem=A)  # set_jacobian + assemble
            mark(7)
        else:  # contract path: A from J, M from H (GN_IN_FULL: lifted gather fused)
            ev_k.record(stream)
            ks.wait_event(ev_k)
            mark(6, ks)
            kkt.set_jacobian(J, mem=A | GN_IN_FULL)
            kkt.assemble(H, dsx, dss, dw_reg, dc_reg, mem=A | GN_IN_FULL)
            mark(7, ks)
            ev_k.record(ks)
            stream.wait_event(ev_k)
        mark(5)

    clocks = Clocks(local_rank)  # sampling from warm-up on; the timed window is selected below
    for _ in range(args.warmup):
        step()
    assert nlp.status(), f"evaluation failed during warm-up: {nlp.last_failure} {nlp.last_error}"
    torch.cuda.synchronize()
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_clk0 = clocks.mark()
    launches0 = L.gn_launch_count()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps, outside the step's events
        step(events[k])
    torch.cuda.synchronize()
    launches = L.gn_launch_count() - launches0
    if dist:
        dist.barrier()
    clk = clocks.stop(t_clk0, clocks.mark())
    assert nlp.status(), "evaluation failed in the timed region"
    per_step = np.array([ev[0].elapsed_time(ev[5]) for ev in events])  # ms
    spans = {"f": (0, 1), "grad+g": (1, 2), "jac": (2, 3), "hess": (3, 4),
             "kkt (set_jacobian + assemble)": (6, 7), "callbacks": (0, 4)}
    per_stage = {k: float(np.mean([ev[a].elapsed_time(ev[b]) for ev in events]))
                 for k, (a, b) in spans.items()}
    ms = float(per_step.mean())
    eager_ms = ms
    # ---- CUDA graph (one graph per unit of work on device-resident
    # buffers).  The whole step -- both streams, fork/join events included -- is
    # captured once and replayed; this is the production launch mode and `value`.
    graph_mode = args.graph and halo is None  # the NCCL halo stays eager; the peer halo is captured
    if graph_mode:
        graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=stream):
            step()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        t_clk0 = clocks.mark()
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                gev[k][0].record(stream)
                graph.replay()
                gev[k][1].record(stream)
        torch.cuda.synchronize()
        clk = clocks.stop(t_clk0, clocks.mark())
        clocks.close()
        assert nlp.status(), "evaluation failed in the graph-timed region"
        ms = float(np.mean([a.elapsed_time(b) for a, b in gev]))
    clocks.close()
    if dist:
        import torch.distributed as tdist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    nnz_rank = s.jac_nnz + s.hess_nnz + kkt.m_nnz
    nnz_step = nnz_rank  # summed over ranks (shards differ by their ghost rows / columns)
    if dist:
        import torch.distributed as tdist
        tt_ = torch.tensor([float(nnz_rank)], dtype=torch.float64, device=dev)
        tdist.all_reduce(tt_)
        nnz_step = int(tt_.item())
    value = nnz_step / (ms * 1e-3)

    # roofline of the dominant kernel: per-kernel CUDA events on the launch stream
    # (library KTimer), measured over extra steps after the timed region
    peak, peak_kind = peaks()
    kkt.set_grid_cap(0)  # standalone per-kernel times: each kernel alone, full grid
    kprof = profile_kernels(L, step, max(3, min(args.steps, 10)), stream, flush)
    kkt.set_grid_cap(grid_cap)
    kb = kernel_bytes(s, kkt, nlp, net, T_rank)
    dom = max(kprof, key=lambda k: kprof[k][0] * kprof[k][1])
    dom_ms = kprof[dom][0]
    achieved = kb.get(dom, 0.0) / (dom_ms * 1e-3) / 1e9
    kernels = {k: {"ms": v[0], "launches_per_step": v[1] / max(3, min(args.steps, 10)),
                   "gbs": kb.get(k, 0.0) / (v[0] * 1e-3) / 1e9 if k in kb else None}
               for k, v in sorted(kprof.items(), key=lambda kv: -kv[1][0] * kv[1][1])}
    unit_bytes = alg_bytes(s, kkt)
    unit_gbs = unit_bytes / (ms * 1e-3) / 1e9

    # line-search trial point: f and g only, one call (gn_eval_fg)
    tev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(0 if args.no_trial else 10)]
    for a_, b_ in tev:
        with torch.cuda.stream(stream):
            flush.zero_()
            a_.record(stream)
            nlp.eval_device("fg", dx, (f, g), sync=False)
            b_.record(stream)
    torch.cuda.synchronize()
    assert nlp.status()
    trial_ms = float(np.median([a_.elapsed_time(b_) for a_, b_ in tev])) if tev else float("nan")
    trial_bytes = 8 * (s.n_vars + s.n_cons + 1)  # x read once, g and f written once
    trial = {"ms": trial_ms, "alg_bytes": trial_bytes,
             "gbs": trial_bytes / (trial_ms * 1e-3) / 1e9,
             "frac": trial_bytes / (trial_ms * 1e-3) / 1e9 / peak}

    ipm_ops = None if args.no_ipm_ops else ipm_vector_ops(nlp, kkt, J, grad, g, dsx, dss, flush,
                                                          stream, peak)

    # ---------------------------------------------------------- e2e (host data)
    # (1) e2e: a device-resident IPM's iteration seen from the host.  Every step
    # copies its inputs (x, w, Sigma_x, Sigma_s) from pinned host memory, runs the
    # same device work as the timed step through the C-ABI (device pointers), and
    # reads back what the host-side solver consumes: f, grad, g and the KKT
    # values A and M.  (2) e2e_contract: the reference's NlpProblem/CondensedKkt
    # seams verbatim -- host spans for x, J, H, A, M on every call (the drop-in
    # integration of INTEGRATION.md), i.e. the J and H round trips included.
    e2e = e2e_contract = None
    if not args.no_e2e:
        pin = lambda k: torch.empty(k, dtype=torch.float64, pin_memory=True)  # noqa
        tx, tw, tsx, tss = pin(s.n_vars), pin(s.n_cons), pin(s.n_free), pin(s.n_cons)
        tx.copy_(torch.from_numpy(x)); tw.copy_(torch.from_numpy(w))
        tsx.copy_(torch.from_numpy(sx)); tss.copy_(torch.from_numpy(ss))
        tf, tgrad, tg = pin(1), pin(s.n_vars), pin(s.n_cons)
        tA, tM = pin(kkt.a_nnz), pin(kkt.m_nnz)
        copy_s = torch.cuda.Stream(device=dev)  # Sigma host -> device beside the callbacks
        d2h_s = torch.cuda.Stream(device=dev)   # f, grad, g device -> host beside the KKT
        ev_sig, ev_cbdone, ev_d2h, ev_vals = (torch.cuda.Event() for _ in range(4))

        def e2e_fused_step():
            # PCIe is full duplex: x and w go first (the callbacks need only them), Sigma
            # follows on a copy stream while the callbacks run (the KKT waits for it), and
            # f, grad, g return while the KKT runs; A and M return after the assembly.
            with torch.cuda.stream(stream):
                dx.copy_(tx, non_blocking=True)
                dwt.copy_(tw, non_blocking=True)
            kw = None
            if world == 1:
                copy_s.wait_stream(stream)  # also orders the reuse of dsx / dss after the last step
                with torch.cuda.stream(copy_s):
                    dsx.copy_(tsx, non_blocking=True)
                    dss.copy_(tss, non_blocking=True)
                ev_sig.record(copy_s)
                kw = ev_sig
            else:  # the halo exchange at the start of the step reads / writes Sigma_s
                with torch.cuda.stream(stream):
                    dsx.copy_(tsx, non_blocking=True)
                    dss.copy_(tss, non_blocking=True)

            def after_cb():
                ev_cbdone.record(stream)
                d2h_s.wait_event(ev_cbdone)
                with torch.cuda.stream(d2h_s):
                    tf.copy_(f, non_blocking=True)
                    tgrad.copy_(grad, non_blocking=True)
                    tg.copy_(g, non_blocking=True)
                ev_d2h.record(d2h_s)

            step(kkt_wait=kw, after_cb=after_cb)
            kkt.values_device(tA, tM, sync=False)  # on the KKT's stream, after the assembly
            ev_vals.record(kstream)
            stream.wait_event(ev_vals)  # the step ends when every copy has landed
            stream.wait_event(ev_d2h)

        class _DevView:  # a zero-copy torch view of a library-owned device array
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                                 "data": (ptr, False), "version": 3}

        pa, pm = kkt.values_ptr()
        vA = torch.as_tensor(_DevView(pa, kkt.a_nnz), device=dev)
        vM = torch.as_tensor(_DevView(pm, kkt.m_nnz), device=dev)
        ev_x2, ev_w, ev_a, ev_fg, ev_m = (torch.cuda.Event() for _ in range(5))

        def e2e_split_step():
            # One GPU: the copies ordered by what each result needs.  x goes up first; A
            # (set_jacobian_x) needs nothing else, so its 0.64 GB start back while w and Sigma
            # go up beside it (PCIe is full duplex) and the callbacks run; f, grad, g follow
            # A back, and M (assemble_x: x, w, Sigma) last.  The device->host stream is busy
            # from the first kernel on.  Same calls and outputs as the timed step, split at
            # the C-ABI's set_jacobian_x / assemble_x seam (gn_kkt_update_x = both).
            with torch.cuda.stream(stream):
                dx.copy_(tx, non_blocking=True)
            ev_x2.record(stream)
            copy_s.wait_stream(stream)  # also orders the reuse of w / Sigma after the last step
            with torch.cuda.stream(copy_s):
                dwt.copy_(tw, non_blocking=True)
                ev_w.record(copy_s)
                dsx.copy_(tsx, non_blocking=True)
                dss.copy_(tss, non_blocking=True)
                ev_sig.record(copy_s)
            kstream.wait_event(ev_x2)
            kkt.set_jacobian_x(dx, mem=A)
            ev_a.record(kstream)
            d2h_s.wait_event(ev_a)
            with torch.cuda.stream(d2h_s):
                tA.copy_(vA, non_blocking=True)
            nlp.eval_device("f", dx, f, sync=False)
            nlp.eval_device("grad", dx, grad, sync=False)
            nlp.eval_device("g", dx, g, sync=False)
            ev_fg.record(stream)
            d2h_s.wait_event(ev_fg)
            with torch.cuda.stream(d2h_s):
                tf.copy_(f, non_blocking=True)
                tgrad.copy_(grad, non_blocking=True)
                tg.copy_(g, non_blocking=True)
            nlp.eval_device("jac", dx, J, sync=False)
            stream.wait_event(ev_w)
            nlp.eval_device("hess", dx, H, w=dwt, ow=1.0, sync=False)
            kstream.wait_event(ev_sig)
            kkt.assemble_x(dx, dwt, 1.0, dsx, dss, dw_reg, dc_reg, mem=A)
            ev_m.record(kstream)
            d2h_s.wait_event(ev_m)
            with torch.cuda.stream(d2h_s):
                tM.copy_(vM, non_blocking=True)
            ev_d2h.record(d2h_s)
            stream.wait_event(ev_d2h)  # the step ends when every copy has landed

        def timed(fn, k):
            fn()
            if dist:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(k):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            t_ms = e0.elapsed_time(e1) / k
            if dist:
                import torch.distributed as tdist
                tt_ = torch.tensor([t_ms], dtype=torch.float64, device=dev)
                tdist.all_reduce(tt_, op=tdist.ReduceOp.MAX)
                t_ms = float(tt_.item())
            return t_ms

        ksteps = max(1, min(args.steps, args.e2e_steps))
        if fused:
            kkt.set_stream(kstream.cuda_stream if world == 1 else stream.cuda_stream)
            e_ms = timed(e2e_split_step if world == 1 else e2e_fused_step, ksteps)
            kkt.set_stream(stream.cuda_stream)
            assert nlp.status()
            # the host copies of the last step are the device results, bit for bit
            dA = torch.empty(kkt.a_nnz, **f64)
            dM = torch.empty(kkt.m_nnz, **f64)
            kkt.values_device(dA, dM, sync=True)
            torch.cuda.synchronize()
            assert torch.equal(tA.to(dev), dA) and torch.equal(tM.to(dev), dM), "e2e A/M copies"
            assert torch.equal(tg.to(dev), g) and torch.equal(tgrad.to(dev), grad), "e2e g/grad"
            assert torch.equal(tf.to(dev), f), "e2e f"
            del dA, dM
            h2d = 8 * (s.n_vars + 2 * s.n_cons + s.n_free)
            d2h = 8 * (1 + s.n_vars + s.n_cons + kkt.a_nnz + kkt.m_nnz)
            e2e = {"value": nnz_step / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": e_ms,
                   "steps": ksteps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                   "path": ("pinned host x, w, Sigma -> device; C-ABI device-pointer calls "
                            "(callbacks + fused KKT, as the timed step); f, grad, g, A, M -> "
                            "pinned host; " + ("x up first, A (set_jacobian_x) back while w "
                                               "and Sigma go up, then f, grad, g, then M "
                                               "(assemble_x)" if world == 1 else
                                               "Sigma in and f, grad, g out overlap the "
                                               "compute"))}

        hx, hw, hsx, hss = tx.numpy(), tw.numpy(), tsx.numpy(), tss.numpy()
        hf, hgrad, hg = tf.numpy(), tgrad.numpy(), tg.numpy()
        hJ, hH = pin(s.jac_nnz).numpy(), pin(s.hess_nnz).numpy()
        hA, hM = tA.numpy(), tM.numpy()
        kkt.set_stream(stream.cuda_stream)

        def e2e_contract_step():
            assert nlp.eval_f(hx, out=hf)[0]
            assert nlp.eval_grad(hx, out=hgrad)[0]
            assert nlp.eval_g(hx, out=hg)[0]
            assert nlp.eval_jac(hx, out=hJ)[0]
            assert nlp.eval_hess(hx, hw, 1.0, out=hH)[0]
            kkt.set_jacobian(hJ, mem=GN_MEM_HOST | GN_IN_FULL)
            kkt.assemble(hH, hsx, hss, dw_reg, dc_reg, mem=GN_MEM_HOST | GN_IN_FULL)
            kkt.values(hA, hM)

        c_ms = timed(e2e_contract_step, ksteps)
        h2d = 8 * (5 * s.n_vars + s.n_cons + s.jac_nnz + s.hess_nnz + s.n_free + s.n_cons)
        d2h = 8 * (1 + s.n_vars + s.n_cons + s.jac_nnz + s.hess_nnz + kkt.a_nnz + kkt.m_nnz)
        e2e_contract = {"value": nnz_step / (c_ms * 1e-3), "unit": UNIT, "ms_per_step": c_ms,
                        "steps": ksteps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "path": "C-ABI GN_MEM_HOST calls (pinned host buffers), "
                                "NlpProblem/CondensedKkt-style (J, H round trips)"}
        if e2e is None:
            e2e = e2e_contract

    # -------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(args.config, args.periods, budget_s=args.cpu_budget, steps=1,
                            warmup=0)
    dropin = None
    if rank == 0 and world == 1 and args.dropin:
        dropin = dropin_ipm()
    seam = None
    if rank == 0 and world == 1 and not args.no_seam:
        seam = dropin_seam(raw, net, scale)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": (f"{args.config} x {args.periods} periods"
                                + (f", period-sharded over {world} GPUs" if args.strong
                                   else " per GPU")
                                + f" (BASELINE configs[{CONFIG_INDEX.get(args.config, '-')}]; "
                                  f"{s.n_vars} vars on rank 0)"),
                   "network": {"buses": net.n_bus, "lines": net.n_line, "gens": net.n_gen,
                               "loads": net.n_load},
                   "periods_per_gpu": T_rank, "periods_total": T_total,
                   "parallelism": f"period-shard x{world}",
                   "halo": None if world == 1 else (f"{halo_kind}: " + (
                       "gn_halo peer-memory stores over NVLink, one kernel per exchange, in "
                       "the CUDA graph" if peer is not None else
                       "torch.distributed NCCL point-to-point, eager" if halo_kind == "nccl"
                       else "gloo, staged through host memory (functional check only)")),
                   "nnz_per_step_per_gpu": {"J": s.jac_nnz, "H": s.hess_nnz, "M": kkt.m_nnz},
                   "l2": "256 MB buffer rewritten between timed steps (outside step events); "
                         "per-step working set ~5.8 GB >> 126 MB L2",
                   "delta_w": dw_reg, "delta_c": dc_reg},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "alg_bytes_per_launch": kb.get(dom), "ms_per_launch": dom_ms,
                     "traffic": None},
        "kernels": kernels,
        "unit_roofline": {"alg_bytes": unit_bytes, "achieved": unit_gbs, "peak": peak,
                          "frac": unit_gbs / peak, "unit": "GB/s"},
        "pipeline": (("fused: set_jacobian/assemble recompute J/H terms from x "
                      "(bit-identical to the contract path, tested)") if fused else
                     "contract: set_jacobian(J) + assemble(H) read the callback outputs")
                    + (f"; {args.streams} streams"),
        "stages_ms": per_stage,
        "line_search_trial": trial,
        "ipm_vector_ops": ipm_ops,
        "launch": (("cuda_graph (eager step %.4f ms)" % eager_ms) if graph_mode else "eager")
        + "; KKT grid cap %d CTA/SM" % grid_cap,
        "setup_s": setup_s,
        "clocks": clk,
        "e2e": e2e,
        "e2e_contract": e2e_contract,
        "cpu_baseline": cpu,
        "dropin_ipm": dropin,
        "dropin_seam": seam,
        "libraries_loaded": loaded_libraries(),
    }
    if args.traffic_json and Path(args.traffic_json).exists():
        tr = json.loads(Path(args.traffic_json).read_text())
        key = dom.split("<")[0] if dom not in tr else dom
        line["roofline"]["traffic"] = tr.get(dom, tr.get(key))
        # measured DRAM bytes of the whole step: ncu bytes per launch x launches per step
        # (the bus3 classes are "k_fz_bus3" and "k_fz_bus3 #2" in the capture)
        if world == 1 and args.config == CONFIG and T_rank == PERIODS_PER_RANK:
            dram = sum(v for k, v in tr.items())
            line["unit_roofline"].update(
                dram_bytes=dram, dram_achieved=dram / (ms * 1e-3) / 1e9,
                dram_frac=dram / (ms * 1e-3) / 1e9 / peak,
                dram_source=f"{_rel(args.traffic_json)} (ncu --set full, per launch; one "
                            f"launch per kernel per step)")
    if rank == 0:
        print(json.dumps(line), flush=True)


def _rel(path) -> str:
    """A path relative to the repository root when it is inside it."""
    try:
        return str(Path(path).resolve().relative_to(ROOT.resolve()))
    except ValueError:
        return str(path)


# ------------------------------------------------------------- reference CPU
def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def loaded_libraries():
    """In-tree / torch-extension shared objects mapped into this process (proof of which
    native code a run used)."""
    out = set()
    try:
        for line in Path("/proc/self/maps").read_text().splitlines():
            path = line.split()[-1] if "/" in line else ""
            if path.endswith(".so") and (path.startswith(str(ROOT)) or "torch_extensions" in path):
                out.add(str(Path(path).relative_to(ROOT)) if path.startswith(str(ROOT)) else path)
    except OSError:
        pass
    return sorted(out)


def _pairs(jr_lifted, m):
    """A^T A row-pair count sum_r len(len+1)/2 (condensed.hpp:55-60) from lifted J rows."""
    c = np.bincount(jr_lifted, minlength=m).astype(np.int64)
    return int((c * (c + 1) // 2).sum())


def cpu_reference(config, periods, budget_s=60.0, steps=None, warmup=1, kkt_periods=8,
                  single_thread=False):
    """The reference's own CPU path (oracle/_ref: the unmodified headers compiled with the
    reference's Release flags) on the box's host cores, at the bench configuration itself.

    * Callbacks at the FULL config: `PatternModel::evaluate_{objective,gradient,constraints}`
      plus `LiftedProblem::eval_jac/eval_hess` (the full callback + pick gather the IPM runs,
      lifted.hpp:128-159), `set_threads(nproc)` (pattern_model.hpp:273); optionally one
      unit at `set_threads(1)`.  Output buffers are allocated once, as IpmSolver does.
    * `CondensedKkt::set_jacobian` + `assemble` (single-threaded by design): the ctor runs
      AMD + a symbolic LDL^T (ldlt.hpp:34-50) that is intractable inside a bench at 15M
      variables, so they are timed on 2- and `kkt_periods`-period windows of the same
      network and extrapolated per contribution (set_jacobian: J_l entries; assemble:
      H_l + A^T A pairs + n_l), SURVEY §8(d).  M nnz at the full horizon is affine in T
      (every coupling but ramp is per period), fitted from the two windows.
    The demand table is the reference's own generate_load_profile (gnr_load_profile): no
    code of this repository's CUDA library is loaded on this path."""
    from oracle import bindings as B
    from paper_2405_14032_b200.network import config_case
    if not B.ref_available():
        return cpu_port(config, budget_s)
    nthreads = os.cpu_count() or 1
    raw = config_case(config, seed=1)
    text = raw.to_matpower()
    scale = B.ref_load_profile(text, periods)
    t0 = time.perf_counter()
    M = B.RefModel(text, periods, scale)
    M.set_threads(nthreads)
    n, m, nj, nh = M.sizes[:4]
    lift = M.lift(1e-4)
    build_s = time.perf_counter() - t0
    nl, _, njl, nhl = M.lifted_sizes
    xl, xu, xs, _, _ = M.bounds()
    x, w, sx, ss = inputs((xl, xu, xs), m, nl)
    del xl, xu, xs
    xfree = np.ascontiguousarray(x[lift["free_to_full"]])
    P = _pairs(lift["jac_rows"], m)
    del lift
    L, h = M.L, M.h
    f = np.zeros(1)
    grad, g, jl, hl = np.empty(n), np.empty(m), np.empty(njl), np.empty(nhl)
    fail = np.zeros(2, np.int32)
    fx, fw, fxf = B._f(x), B._f(w), B._f(xfree)

    def callbacks():
        assert L.gnr_eval_f(h, fx, B._f(f), B._i(fail))
        assert L.gnr_eval_grad(h, fx, B._f(grad), B._i(fail))
        assert L.gnr_eval_g(h, fx, B._f(g), B._i(fail))
        assert L.gnr_lifted_eval_jac(h, fxf, B._f(jl))
        assert L.gnr_lifted_eval_hess(h, fxf, fw, 1.0, B._f(hl))

    for _ in range(warmup):
        callbacks()
    times = []
    t_start = time.perf_counter()
    while True:
        a = time.perf_counter()
        callbacks()
        times.append(time.perf_counter() - a)
        if steps is not None and len(times) >= steps:
            break
        if time.perf_counter() - t_start > budget_s:
            break
    cb_s = float(np.median(times))
    cb1_s = None
    if single_thread:
        M.set_threads(1)
        a = time.perf_counter()
        callbacks()
        cb1_s = time.perf_counter() - a
        M.set_threads(nthreads)
    del grad, g, jl, hl, M

    # condensed KKT on period windows of the same network
    wins = sorted({min(2, periods), min(kkt_periods, periods)})
    kw = []
    for Tw in wins:
        W = B.RefModel(text, Tw, scale[:Tw])
        lw = W.lift(1e-4)
        nlw, mw, njw, nhw = W.lifted_sizes
        Pw = _pairs(lw["jac_rows"], mw)
        dims = W.kkt_create()
        xw, ww, sxw, ssw = inputs(W.bounds()[:3], mw, nlw)
        jw, hw = np.empty(njw), np.empty(nhw)
        assert W.L.gnr_lifted_eval_jac(W.h, B._f(np.ascontiguousarray(xw[lw["free_to_full"]])),
                                       B._f(jw))
        assert W.L.gnr_lifted_eval_hess(W.h, B._f(np.ascontiguousarray(xw[lw["free_to_full"]])),
                                        B._f(ww), 1.0, B._f(hw))
        sj, sa = [], []
        for _ in range(3):
            a = time.perf_counter()
            W.kkt_set_jacobian(jw)
            b = time.perf_counter()
            W.kkt_assemble(hw, sxw, ssw, 1e-4, 1e-8 * 0.1 ** 0.25)
            sj.append(b - a)
            sa.append(time.perf_counter() - b)
        kw.append(dict(periods=Tw, set_jacobian_ms=1e3 * float(np.median(sj)),
                       assemble_ms=1e3 * float(np.median(sa)), jac_lifted=njw,
                       assemble_contributions=nhw + Pw + nlw, m_nnz=int(dims[2]),
                       ns_per_jac=1e9 * float(np.median(sj)) / max(njw, 1),
                       ns_per_contribution=1e9 * float(np.median(sa)) / max(nhw + Pw + nlw, 1)))
        del W
    big = kw[-1]
    if big["periods"] == periods:  # measured at the full horizon: no extrapolation
        kkt_s = 1e-3 * (big["set_jacobian_ms"] + big["assemble_ms"])
        mnnz = big["m_nnz"]
        kkt_kind = "measured"
    else:
        kkt_s = 1e-9 * (big["ns_per_jac"] * njl + big["ns_per_contribution"] * (nhl + P + nl))
        a0, a1 = kw[0], kw[-1]  # M nnz affine in T
        slope = (a1["m_nnz"] - a0["m_nnz"]) / (a1["periods"] - a0["periods"])
        mnnz = int(round(a1["m_nnz"] + slope * (periods - a1["periods"])))
        kkt_kind = "extrapolated"
    t_unit = cb_s + kkt_s
    nnz = nj + nh + mnnz
    return {"value": nnz / t_unit, "unit": UNIT, "cores": nthreads, "kind": "reference",
            "cpu_model": cpu_model(), "same_config": True, "ms_per_unit": t_unit * 1e3,
            "callbacks_ms": cb_s * 1e3, "callbacks_ms_1thread": None if cb1_s is None else cb1_s * 1e3,
            "kkt_ms": kkt_s * 1e3, "kkt": kkt_kind, "kkt_windows": kw,
            "units_timed": len(times), "build_s": build_s,
            "nnz_per_unit": {"J": nj, "H": nh, "M": mnnz},
            "sample": f"{config} x {periods} periods, the bench configuration itself (n={n}, "
                      f"J={nj}, H={nh}): callbacks (f, grad, g, lifted jac + hess) with "
                      f"PatternModel::set_threads({nthreads}), median of {len(times)} units; "
                      f"CondensedKkt set_jacobian + assemble (single-threaded by design) "
                      f"{kkt_kind} from {'/'.join(str(k['periods']) for k in kw)}-period "
                      f"windows per contribution (J_l={njl}, H_l + pairs + n_l = "
                      f"{nhl + P + nl}; M={mnnz})"}


def cpu_port(config, budget_s=15.0, periods=2):
    """Without oracle/_ref (no /root/reference at build time): the C restatement
    (oracle/gn_oracle.c, single-threaded) on a `periods`-period sample."""
    from oracle import bindings as B
    from paper_2405_14032_b200.network import config_case
    raw = config_case(config, seed=1)
    net = raw.network()
    scale = np.ones((periods, net.n_load))
    Mo = B.OracleModel(net, periods, scale)
    xl, xu, xs, _, _ = Mo.bounds()
    n, m, nj, nh = Mo.sizes[:4]
    lift = Mo.lift(1e-4)
    x, w, sx, ss = inputs((xl, xu, xs), m, len(lift["free_to_full"]))
    K = Mo.kkt()
    times = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and len(times) < 50:
        a = time.perf_counter()
        assert Mo.eval_f(x)[0] and Mo.eval_grad(x)[0] and Mo.eval_g(x)[0]
        _, jv, _ = Mo.eval_jac(x)
        _, hv, _ = Mo.eval_hess(x, w, 1.0)
        K.set_jacobian(jv[lift["jac_pick"]])
        K.assemble(hv[lift["hess_pick"]], sx, ss, 1e-4, 1e-8 * 0.1 ** 0.25)
        times.append(time.perf_counter() - a)
    t_unit = float(np.median(times))
    return {"value": (nj + nh + K.m_nnz) / t_unit, "unit": UNIT, "cores": 1, "kind": "port",
            "cpu_model": cpu_model(), "same_config": False, "ms_per_unit": t_unit * 1e3,
            "units_timed": len(times),
            "sample": f"{config} network x {periods} periods (unit demand scale), C restatement "
                      f"(oracle/gn_oracle.c), one thread"}


def dropin_seam(raw, net, scale, units=3):
    """The hot-path unit through the reference's own seams (oracle/_ref/seam_bench): the
    LiftedProblem and CondensedKkt the IpmSolver builds, over gridnlp_b200::CudaOpfNlp,
    with pageable std::vector spans -- the drop-in integration as a user of the reference
    gets it, at the bench configuration.  Two runs: the shim LiftedProblem (lifted staging
    and J / H gathers on the device, the default) and the reference's own LiftedProblem
    (GRIDNLP_B200_HOST_LIFTED=1: host staging and gathers), the latter as `host_lifted`."""
    import os
    import subprocess
    import tempfile
    from oracle import bindings as B
    exe = B.HERE / "_ref" / "seam_bench"
    if not exe.exists():
        return None

    def one(path, host_lifted):
        env = dict(os.environ, GRIDNLP_B200_HOST_LIFTED="1" if host_lifted else "0")
        out = subprocess.run([str(exe), str(path), "cuda", str(units)], capture_output=True,
                             text=True, timeout=1200, env=env)
        if out.returncode != 0:
            return {"error": out.stderr.strip()[-300:]}
        r = json.loads(out.stdout.strip().splitlines()[-1])
        r["value"] = r["nnz_per_unit"] / (r["ms_per_unit"] * 1e-3)
        r["unit"] = UNIT
        return r

    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "net.bin"
        B.write_network_bin(path, net, scale.shape[0], scale)
        r = one(path, False)
        if "error" in r:
            return r
        r["path"] = ("shim LiftedProblem (device staging + gathers) + CudaOpfNlp lifted calls "
                     "(GN_MEM_HOST) + shim CondensedKkt set_jacobian / assemble, pageable "
                     "std::vector spans")
        h = one(path, True)
        if "error" not in h:
            h = {k: h[k] for k in ("ms_per_unit", "callbacks_ms", "kkt_ms", "value",
                                   "lifted_device")}
            h["path"] = "the reference's own LiftedProblem (host staging + gathers), same rest"
        r["host_lifted"] = h
    return r


def dropin_ipm(periods=24):
    """The UNMODIFIED reference interior-point solver end to end, twice on the same problem
    (synthetic case118-size x `periods`): with the reference's own callbacks and
    CondensedKkt (oracle/_ref, gnr_solve), and through the drop-in seams on the B200 path
    (oracle/_ref/ipm_dropin cuda: CudaOpfNlp + the shadowing CondensedKkt).  The sparse
    LDL^T stays on the host in both (out of scope), so this bounds the end-to-end gain of
    the drop-in at this size; wall seconds of solve_nlp, problem construction excluded."""
    import subprocess
    import tempfile
    from oracle import bindings as B
    from paper_2405_14032_b200.network import config_case
    from paper_2405_14032_b200.opf import load_profile
    if not (B.ref_available() and B.DROPIN.exists()):
        return None
    raw = config_case("case118")
    net = raw.network()
    scale = load_profile(net.n_load, periods)
    model = B.RefModel(raw.to_matpower(), periods, scale)
    refs = [model.solve(1e-4) for _ in range(3)]
    ref = dict(refs[0], seconds=float(np.median([r["seconds"] for r in refs])))
    runs = []
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "net.bin"
        B.write_network_bin(path, net, periods, scale)
        for _ in range(3):
            out = subprocess.run([str(B.DROPIN), str(path), "cuda", "1e-4", "2"],
                                 capture_output=True, text=True, timeout=600)
            if out.returncode != 0:
                return {"error": out.stderr.strip()[-300:]}
            runs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    ours = dict(runs[0], warm_seconds=float(np.median([r["warm_seconds"] for r in runs])))
    return {"case": f"synthetic case118 x {periods} periods", "tol": 1e-4,
            "reference": {"iterations": ref["iterations"], "objective": ref["objective"],
                          "seconds": ref["seconds"]},
            "b200_dropin": {"iterations": ours["iterations"], "objective": ours["objective"],
                            "seconds": ours["warm_seconds"]},
            "objective_rel_diff": abs(ours["objective"] - ref["objective"]) / abs(ref["objective"]),
            "speedup": ref["seconds"] / ours["warm_seconds"]}


def run_reference(args, rank, world):
    """`--impl reference`: the reference's own CPU implementation of the path on this box's
    host cores, at our arm's config / metric / unit (rank 0 only; other ranks exit 0)."""
    if rank != 0:
        return
    cpu = cpu_reference(args.config, args.periods, budget_s=args.cpu_budget,
                        steps=args.steps, warmup=min(args.warmup, 1), single_thread=True)
    line = {
        "metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["ms_per_unit"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.config} x {args.periods} periods "
                               f"(BASELINE configs[{CONFIG_INDEX.get(args.config, '-')}]; the "
                               f"same workload as our arm)",
                   "parallelism": f"host threads ({cpu['cores']})",
                   "timed": f"{cpu['units_timed']} units (wall budget {args.cpu_budget} s; "
                            f"--steps {args.steps} is the cap)"},
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "libraries_loaded": loaded_libraries(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--periods", type=int, default=PERIODS_PER_RANK)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=60.0,
                    help="wall budget (s) of the reference arm's timed callback units")
    ap.add_argument("--pipeline", choices=["fused", "contract"], default="fused")
    ap.add_argument("--streams", type=int, choices=[1, 2], default=2)
    ap.add_argument("--grid-cap", type=int, default=-1,
                    help="KKT CTAs per SM (default: 2 with two streams, else uncapped)")
    ap.add_argument("--dropin", action="store_true",
                    help="also time whole reference-IPM solves, reference vs drop-in (host-"
                         "LDL^T-bound, noisy: median of 3 each)")
    ap.add_argument("--no-dropin", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-seam", action="store_true",
                    help="skip the drop-in seam timing (oracle/_ref/seam_bench)")
    ap.add_argument("--no-trial", action="store_true",
                    help="skip the line-search trial (gn_eval_fg) measurement")
    ap.add_argument("--no-ipm-ops", action="store_true",
                    help="skip the device-resident IPM vector-op measurement")
    ap.add_argument("--graph", type=int, choices=[0, 1], default=1,
                    help="replay the step as one CUDA graph (with the peer halo under torchrun)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: --periods is the whole horizon, partitioned over the "
                         "ranks (e.g. configs[3]: --config case13659pegase --periods 168)")
    ap.add_argument("--halo", choices=["peer", "nccl", "gloo"], default="peer",
                    help="period-shard halo: peer-memory stores (gn_halo) or NCCL p2p")
    ap.add_argument("--traffic-json", default=str(ROOT / "profiles" / "traffic.json"))
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist = None
    # GN_BENCH_ONE_GPU=1: a functional check of the multi-rank path on one GPU -- every rank on
    # cuda:0, a gloo group, the halo staged through host memory (no kernel waits on another
    # process's kernel); its timings mean nothing
    one_gpu = world > 1 and os.environ.get("GN_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
        args.halo = "gloo"
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        if one_gpu:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    try:
        run_ours(args, rank, world, local_rank, dist)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
