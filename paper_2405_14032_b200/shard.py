"""Period sharding of the multi-period OPF — host-side logic.

The horizon [0, T_total) is split into contiguous period ranges, one per rank.
Rank r's device problem (gn_ctx_create_shard) is the reference layout
(power/opf.hpp:16-60) over its own periods plus ghost generator set-points:

* ghost_prev[k] = pg(ramp_gen k, t0 - 1): fixed, filled with rank r-1's value;
* ghost_next[k] = pg(ramp_gen k, t1):     free; it appears only in the ramp rows
  of step t1, which rank r carries as *ghost rows* (owned by rank r+1, whose
  sigma_s values rank r receives).

The ramp row of step t belongs to the rank that owns period t.  With the halo
filled, every owned row value, Jacobian/Hessian record and lifted M column of
a shard equals the global problem's, bit for bit (tests/test_shard.py).  The
only exchanges per IPM iteration are G-sized: the boundary set-points
(forward and backward) and the sigma_s of the boundary ramp rows (backward).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition(T_total: int, world: int) -> list[tuple[int, int]]:
    """Contiguous (first_period, periods) per rank; the first T_total % world ranks get one more."""
    if world < 1 or T_total < world:
        raise ValueError("need at least one period per rank")
    base, extra = divmod(T_total, world)
    out, t0 = [], 0
    for r in range(world):
        T = base + (1 if r < extra else 0)
        out.append((t0, T))
        t0 += T
    return out


@dataclass
class Layout:
    """OpfLayout offsets for a horizon of T periods (opf.hpp:135-230)."""
    N: int
    L: int
    G: int
    LT: int
    GR: int
    T: int
    R: int      # ramp rows per ramp generator
    s_lo: int   # first ramp step

    @property
    def var_blocks(self):  # (offset, count) of pg, qg, p, q, v, th
        G, L, N, T = self.G, self.L, self.N, self.T
        offs = np.cumsum([0, G * T, G * T, L * T, L * T, N * T])
        return list(zip(offs.tolist(), [G, G, L, L, N, N]))

    @property
    def row_blocks(self):  # bal_p, bal_q, flow_p, flow_q, thermal, angle
        N, L, LT, T = self.N, self.L, self.LT, self.T
        offs = np.cumsum([0, N * T, N * T, L * T, L * T, LT * T])
        return list(zip(offs.tolist(), [N, N, L, L, LT, L]))

    @property
    def n_base(self):
        return 2 * self.T * (self.G + self.L + self.N)

    @property
    def ramp0(self):
        return (2 * self.N + 3 * self.L + self.LT) * self.T


class ShardMap:
    """Local <-> global index maps of rank r's shard [t0, t0 + T)."""

    def __init__(self, N: int, L: int, G: int, LT: int, ramp_gens, T_total: int, t0: int, T: int):
        self.ramp_gens = np.asarray(ramp_gens, np.int64)
        GR = len(self.ramp_gens) if T_total >= 2 else 0
        self.T_total, self.t0, self.T = T_total, t0, T
        self.prev, self.next = t0 > 0, t0 + T < T_total
        self.glob = Layout(N, L, G, LT, GR, T_total, max(T_total - 1, 0), 1)
        self.loc = Layout(N, L, G, LT, GR, T, T - 1 + self.prev + self.next, 0 if self.prev else 1)
        self.GR = GR

    # ------------------------------------------------------------- variables
    @property
    def n_local(self):
        return self.loc.n_base + self.GR * (self.prev + self.next)

    def var_global(self) -> np.ndarray:
        """Global index of every local variable (ghosts included)."""
        out = []
        t = np.arange(self.T)
        for (lo, cnt), (go, _) in zip(self.loc.var_blocks, self.glob.var_blocks):
            e = np.arange(cnt)[:, None]
            out.append((go + e * self.T_total + self.t0 + t[None, :]).reshape(-1))
        if self.prev:
            out.append(self.ramp_gens * self.T_total + self.t0 - 1)
        if self.next:
            out.append(self.ramp_gens * self.T_total + self.t0 + self.T)
        return np.concatenate(out).astype(np.int64)

    def ghost_prev(self) -> np.ndarray:
        return np.arange(self.GR) + self.loc.n_base if self.prev else np.zeros(0, np.int64)

    def ghost_next(self) -> np.ndarray:
        start = self.loc.n_base + (self.GR if self.prev else 0)
        return np.arange(self.GR) + start if self.next else np.zeros(0, np.int64)

    # ------------------------------------------------------------------ rows
    def ramp_steps(self) -> np.ndarray:
        return np.arange(self.loc.s_lo, self.loc.s_lo + self.loc.R)

    @property
    def m_local(self):
        return self.loc.ramp0 + self.GR * self.loc.R

    def row_global(self) -> np.ndarray:
        out = []
        t = np.arange(self.T)
        for (lo, cnt), (go, _) in zip(self.loc.row_blocks, self.glob.row_blocks):
            e = np.arange(cnt)[:, None]
            out.append((go + e * self.T_total + self.t0 + t[None, :]).reshape(-1))
        if self.GR and self.loc.R > 0:
            k = np.arange(self.GR)[:, None]
            step = self.t0 + self.ramp_steps()[None, :]  # global step t
            out.append((self.glob.ramp0 + k * self.glob.R + step - 1).reshape(-1))
        return np.concatenate(out).astype(np.int64) if out else np.zeros(0, np.int64)

    def row_owned(self) -> np.ndarray:
        """Ramp rows of step t1 (local step T) are ghosts owned by the next rank."""
        own = np.ones(self.m_local, bool)
        if self.next and self.GR:
            k = np.arange(self.GR)
            own[self.loc.ramp0 + k * self.loc.R + (self.T - self.loc.s_lo)] = False
        return own

    # ------------------------------------------------------------------ halo
    def first_ramp_rows(self) -> np.ndarray:
        """Local rows of step t0 (the boundary rows this rank owns when prev)."""
        k = np.arange(self.GR)
        return self.loc.ramp0 + k * self.loc.R if self.prev else np.zeros(0, np.int64)

    def ghost_rows(self) -> np.ndarray:
        k = np.arange(self.GR)
        return (self.loc.ramp0 + k * self.loc.R + (self.T - self.loc.s_lo)) if self.next \
            else np.zeros(0, np.int64)

    def pg_first(self) -> np.ndarray:
        """Local indices of pg(ramp gen k, first period) — sent to the previous rank."""
        return self.ramp_gens * self.T

    def pg_last(self) -> np.ndarray:
        """Local indices of pg(ramp gen k, last period) — sent to the next rank."""
        return self.ramp_gens * self.T + self.T - 1

    def halo_plan(self, device=None) -> dict:
        """Index tensors of the distributed exchange (exchange_halo)."""
        import torch
        ix = lambda a: torch.from_numpy(np.asarray(a, np.int64)).to(device)  # noqa: E731
        return dict(pg_last=ix(self.pg_last()), pg_first=ix(self.pg_first()),
                    g_prev=ix(self.ghost_prev()), g_next=ix(self.ghost_next()),
                    rows_first=ix(self.first_ramp_rows()), rows_ghost=ix(self.ghost_rows()),
                    GR=self.GR, prev=self.prev, next=self.next)


def exchange_halo(plan: dict, x, sigma_s, rank: int, stage_cpu: bool = False):
    """One ramp-halo exchange with torch.distributed (NCCL on device tensors in
    bench.py; gloo on CPU in tests/test_shard_gloo.py; `stage_cpu`: device tensors whose
    messages go through host memory, for a gloo group): pg(., t1-1) to the next
    rank, pg(., t0) and the boundary rows' sigma_s to the previous rank, written
    into this rank's ghost set-points / ghost rows.  G doubles per message."""
    import torch
    import torch.distributed as tdist
    kw = dict(dtype=x.dtype, device="cpu" if stage_cpu else x.device)
    msg = (lambda t: t.cpu()) if stage_cpu else (lambda t: t)  # noqa: E731
    ops, recv = [], {}
    if plan["next"]:
        ops.append(tdist.P2POp(tdist.isend, msg(x.index_select(0, plan["pg_last"])), rank + 1))
        recv["xn"] = torch.empty(plan["GR"], **kw)
        recv["sn"] = torch.empty(plan["GR"], **kw)
        ops.append(tdist.P2POp(tdist.irecv, recv["xn"], rank + 1))
        ops.append(tdist.P2POp(tdist.irecv, recv["sn"], rank + 1))
    if plan["prev"]:
        recv["xp"] = torch.empty(plan["GR"], **kw)
        ops.append(tdist.P2POp(tdist.irecv, recv["xp"], rank - 1))
        ops.append(tdist.P2POp(tdist.isend, msg(x.index_select(0, plan["pg_first"])), rank - 1))
        ops.append(tdist.P2POp(tdist.isend, msg(sigma_s.index_select(0, plan["rows_first"])),
                               rank - 1))
    if ops:
        for wk in tdist.batch_isend_irecv(ops):
            wk.wait()
    if "xp" in recv:
        x.index_copy_(0, plan["g_prev"], recv["xp"].to(x.device))
    if "xn" in recv:
        x.index_copy_(0, plan["g_next"], recv["xn"].to(x.device))
        sigma_s.index_copy_(0, plan["rows_ghost"], recv["sn"].to(x.device))


def global_objective(f_local, world: int):
    """The global problem's objective from the shards' partial objectives:
    all-gather the per-rank partials (one double each) and add them in rank order, so
    every rank holds the same, run-to-run identical value.  (The reference sums the
    records of all periods in one sequence; the rank-order sum of the period-shard
    partials agrees with it to rounding.)  `f_local` is a 1-element tensor on the rank's
    device; returns a 1-element tensor."""
    import torch
    import torch.distributed as tdist
    src = f_local.cpu() if tdist.get_backend() == "gloo" else f_local
    parts = [torch.empty_like(src) for _ in range(world)]
    tdist.all_gather(parts, src)
    total = parts[0].clone()
    for p in parts[1:]:
        total += p
    return total.to(f_local.device)


class DeviceHalo:
    """The period-shard halo over peer memory (gn_halo, csrc/gn_halo.cu): this rank's
    neighbours store the boundary set-points / sigma_s and their objective partials
    straight into a small region of this rank's device memory (NVLink / NVSwitch P2P)
    and release a step flag; one kernel per exchange, no host call, so a step that
    contains the exchanges is capturable in one CUDA graph."""

    SEND, RECV, BOTH = 1, 2, 3
    HANDLE_BYTES = 64

    def __init__(self, nlp, rank: int, world: int):
        import ctypes as C
        from . import abi
        from .opf import _check
        self.lib, self.nlp, self.rank, self.world = abi.lib(), nlp, rank, world
        h, err = C.c_void_p(), abi.GnError()
        _check(self.lib.gn_halo_create(nlp.h, rank, world, C.byref(h), C.byref(err)), err,
               "gn_halo_create")
        self.h = h

    def ipc_handle(self) -> bytes:
        import ctypes as C
        buf = (C.c_ubyte * self.HANDLE_BYTES)()
        self._ok(self.lib.gn_halo_ipc_handle(self.h, buf))
        return bytes(buf)

    def open(self, handles: list[bytes]):
        """Map every other rank's region (handles[q] from rank q, e.g. all_gather_object)."""
        import ctypes as C
        raw = b"".join(handles)
        assert len(raw) == self.HANDLE_BYTES * self.world
        buf = (C.c_ubyte * len(raw)).from_buffer_copy(raw)
        self._ok(self.lib.gn_halo_open(self.h, buf))

    def connect(self):
        """open() with the handles all-gathered over the default process group."""
        import torch.distributed as tdist
        handles = [None] * self.world
        tdist.all_gather_object(handles, self.ipc_handle())
        self.open(handles)

    @staticmethod
    def link(halos: list["DeviceHalo"]):
        """Same process: the ranks' halos (index = rank) see each other's regions."""
        import ctypes as C
        arr = (C.c_void_p * len(halos))(*[x.h.value for x in halos])
        halos[0]._ok(halos[0].lib.gn_halo_link(arr, len(halos)))

    def exchange(self, x, sigma_s, phase: int = 3, stream: int = 0):
        from .opf import _f64
        import ctypes as C
        self._ok(self.lib.gn_halo_exchange(self.h, _f64(x), _f64(sigma_s), phase,
                                           C.c_void_p(stream)))

    def objective(self, f_local, f_global, phase: int = 3, stream: int = 0):
        from .opf import _f64
        import ctypes as C
        self._ok(self.lib.gn_halo_objective(self.h, _f64(f_local), _f64(f_global), phase,
                                            C.c_void_p(stream)))

    @staticmethod
    def exchange_emulated(halos: list["DeviceHalo"], xs, sigma_s, stream: int = 0):
        """All ranks' exchanges in one cooperative launch (one GPU)."""
        import ctypes as C
        from . import abi
        from .opf import _f64
        k = len(halos)
        hs = (C.c_void_p * k)(*[x.h.value for x in halos])
        px = (abi.f64p * k)(*[_f64(a) for a in xs])
        ps = (abi.f64p * k)(*[_f64(a) for a in sigma_s])
        halos[0]._ok(halos[0].lib.gn_halo_exchange_emulated(hs, k, px, ps, C.c_void_p(stream)))

    def close(self):
        if getattr(self, "h", None):
            self.lib.gn_halo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ok(self, rc):
        from .opf import _check
        _check(rc, None, "gn_halo")


def halo_exchange(maps: list[ShardMap], xs: list[np.ndarray], sigma_s: list[np.ndarray]):
    """In-process halo fill (all ranks' arrays at hand): what the distributed
    exchange in bench.py / tests/test_shard_gloo.py does with send/recv."""
    for r, mp in enumerate(maps):
        if mp.prev:
            xs[r][mp.ghost_prev()] = xs[r - 1][maps[r - 1].pg_last()]
        if mp.next:
            xs[r][mp.ghost_next()] = xs[r + 1][maps[r + 1].pg_first()]
            sigma_s[r][mp.ghost_rows()] = sigma_s[r + 1][maps[r + 1].first_ramp_rows()]
