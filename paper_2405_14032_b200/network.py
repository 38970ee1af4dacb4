"""Network data in the reference's per-unit NetworkData form (SoA numpy).

* `Network` mirrors power::NetworkData (power/network.hpp:50-66).
* `RawCase` holds MATPOWER-unit data (MW, degrees, $/MWh) and converts with
  the same floating-point operations as parse_matpower
  (power/matpower.hpp:119-272), so the per-unit arrays are bit-identical to
  what the reference parser produces from `RawCase.to_matpower()` text.
* `synthetic_case` draws ring + chord networks with case118-fixture statistics
  (data/case118.m:2-5) at any size.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from .abi import GnNetwork

K_PI = math.pi  # common.hpp:17 kPi as a double


@dataclass
class Network:
    base_mva: float
    reference_bus: int
    bus_vmin: np.ndarray
    bus_vmax: np.ndarray
    vm_start: np.ndarray
    va_start: np.ndarray
    line_from: np.ndarray
    line_to: np.ndarray
    line_g: np.ndarray
    line_b: np.ndarray
    line_smax: np.ndarray
    line_amin: np.ndarray
    line_amax: np.ndarray
    gen_bus: np.ndarray
    gen_pmin: np.ndarray
    gen_pmax: np.ndarray
    gen_qmin: np.ndarray
    gen_qmax: np.ndarray
    gen_ramp: np.ndarray
    gen_c2: np.ndarray
    gen_c1: np.ndarray
    gen_c0: np.ndarray
    gen_pstart: np.ndarray
    gen_qstart: np.ndarray
    load_bus: np.ndarray
    load_p: np.ndarray
    load_q: np.ndarray
    _keep: list = field(default_factory=list, repr=False)

    F64 = ("bus_vmin", "bus_vmax", "vm_start", "va_start", "line_g", "line_b", "line_smax",
           "line_amin", "line_amax", "gen_pmin", "gen_pmax", "gen_qmin", "gen_qmax",
           "gen_ramp", "gen_c2", "gen_c1", "gen_c0", "gen_pstart", "gen_qstart", "load_p",
           "load_q")
    I32 = ("line_from", "line_to", "gen_bus", "load_bus")

    def __post_init__(self):
        for k in self.F64:
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=np.float64))
        for k in self.I32:
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=np.int32))

    @property
    def n_bus(self) -> int:
        return len(self.bus_vmin)

    @property
    def n_line(self) -> int:
        return len(self.line_from)

    @property
    def n_gen(self) -> int:
        return len(self.gen_bus)

    @property
    def n_load(self) -> int:
        return len(self.load_bus)

    def to_c(self) -> GnNetwork:
        """ctypes gn_network view (arrays stay owned by this object)."""
        s = GnNetwork()
        s.n_bus, s.n_line, s.n_gen, s.n_load = self.n_bus, self.n_line, self.n_gen, self.n_load
        s.reference_bus = self.reference_bus
        for k in self.F64:
            setattr(s, k, getattr(self, k).ctypes.data_as(C.POINTER(C.c_double)))
        for k in self.I32:
            setattr(s, k, getattr(self, k).ctypes.data_as(C.POINTER(C.c_int32)))
        return s

    def equal(self, other: "Network") -> bool:
        if self.reference_bus != other.reference_bus or self.base_mva != other.base_mva:
            return False
        return all(np.array_equal(getattr(self, k), getattr(other, k)) for k in self.F64 + self.I32)


@dataclass
class RawCase:
    """MATPOWER-unit case (the subset parse_matpower accepts)."""
    base_mva: float
    bus: np.ndarray      # [N, 13] bus_i type Pd Qd Gs Bs area Vm Va baseKV zone Vmax Vmin
    gen: np.ndarray      # [G, 10] bus Pg Qg Qmax Qmin Vg mBase status Pmax Pmin
    branch: np.ndarray   # [L, 13] fbus tbus r x b rateA rateB rateC ratio angle status angmin angmax
    gencost: np.ndarray  # [G, 7]  2 startup shutdown 3 c2 c1 c0

    def to_matpower(self) -> str:
        def mat(name, a, ints):
            rows = []
            for r in a:
                cells = [str(int(v)) if j in ints else repr(float(v)) for j, v in enumerate(r)]
                rows.append("\t" + "\t".join(cells) + ";")
            return f"mpc.{name} = [\n" + "\n".join(rows) + "\n];\n"
        return ("function mpc = synthetic\nmpc.version = '2';\n"
                f"mpc.baseMVA = {self.base_mva!r};\n"
                + mat("bus", self.bus, {0, 1, 6, 10})
                + mat("gen", self.gen, {0, 7})
                + mat("branch", self.branch, {0, 1, 10})
                + mat("gencost", self.gencost, {0, 3}))

    def network(self, ramp_fraction: float = 0.1) -> Network:
        """Per-unit conversion with parse_matpower's arithmetic (matpower.hpp:119-272)."""
        base = float(self.base_mva)
        bus, gen, br, gc = self.bus, self.gen, self.branch, self.gencost
        ids = {int(b[0]): i for i, b in enumerate(bus)}
        ref = [i for i, b in enumerate(bus) if int(b[1]) == 3]
        assert len(ref) == 1
        load_rows = [i for i, b in enumerate(bus) if b[2] != 0.0 or b[3] != 0.0]
        g_in = [i for i, g in enumerate(gen) if g[7] > 0.0]
        b_in = [i for i, b in enumerate(br) if b[10] != 0.0]
        pmax = np.array([gen[i][8] / base for i in g_in])
        rr = np.array([br[i][2] for i in b_in])
        xx = np.array([br[i][3] for i in b_in])
        z2 = rr * rr + xx * xx
        amin = np.array([br[i][11] for i in b_in], dtype=np.float64)
        amax = np.array([br[i][12] for i in b_in], dtype=np.float64)
        unset = (amin == 0.0) & (amax == 0.0)
        amin = np.where(unset | (amin <= -360.0), -60.0, amin)
        amax = np.where(unset | (amax >= 360.0), 60.0, amax)
        rate = np.array([br[i][5] for i in b_in])
        c2 = np.array([gc[i][4] for i in g_in])
        c1 = np.array([gc[i][5] for i in g_in])
        c0 = np.array([gc[i][6] for i in g_in])
        return Network(
            base_mva=base, reference_bus=ref[0],
            bus_vmin=bus[:, 12], bus_vmax=bus[:, 11], vm_start=bus[:, 7],
            va_start=bus[:, 8] * K_PI / 180.0,
            line_from=[ids[int(br[i][0])] for i in b_in],
            line_to=[ids[int(br[i][1])] for i in b_in],
            line_g=rr / z2, line_b=-xx / z2,
            line_smax=np.where(rate > 0.0, rate / base, np.inf),
            line_amin=amin * K_PI / 180.0, line_amax=amax * K_PI / 180.0,
            gen_bus=[ids[int(gen[i][0])] for i in g_in],
            gen_pmin=np.array([gen[i][9] / base for i in g_in]), gen_pmax=pmax,
            gen_qmin=np.array([gen[i][4] / base for i in g_in]),
            gen_qmax=np.array([gen[i][3] / base for i in g_in]),
            gen_ramp=(ramp_fraction * np.maximum(pmax, 0.0)) if ramp_fraction < math.inf
            else np.full(len(g_in), np.inf),
            gen_c2=c2 * base * base, gen_c1=c1 * base, gen_c0=c0,
            gen_pstart=np.array([gen[i][1] / base for i in g_in]),
            gen_qstart=np.array([gen[i][2] / base for i in g_in]),
            load_bus=load_rows,
            load_p=np.array([bus[i][2] / base for i in load_rows]),
            load_q=np.array([bus[i][3] / base for i in load_rows]),
        )


# Sizes of the BASELINE.json configurations (N / L / G / D), SURVEY.md §8(d).
CONFIG_SIZES = {
    "case118": (118, 186, 54, 99),
    "case1354pegase": (1354, 1991, 260, 1137),
    "case9241pegase": (9241, 16049, 1445, 7762),
    "case13659pegase": (13659, 20467, 4092, 11473),
    "synthetic30k": (30000, 45000, 4500, 25200),
}


def synthetic_case(n_bus: int, n_line: int, n_gen: int, n_load: int, seed: int = 1,
                   parallel_lines: int = 0, shared_gens: int = 0, max_span: int = 20,
                   load_scale: float = 1.0) -> RawCase:
    """Ring + seeded chords (no self-loops), case118-fixture statistics.

    `parallel_lines` adds that many duplicate-terminal lines and `shared_gens`
    that many extra generators on already-used buses (edge cases for the
    balance-row accumulation order and AtA pattern).  `load_scale` multiplies every
    demand (the BASELINE sizes carry fewer generators per load than case118, so an
    end-to-end solve needs lighter loads to be feasible); the draw is unchanged."""
    assert n_line >= n_bus >= 3 and 1 <= n_gen and n_load <= n_bus
    rng = np.random.default_rng(seed)
    N = n_bus
    # ring
    fr = list(range(N))
    to = [(i + 1) % N for i in range(N)]
    seen = {(min(a, b), max(a, b)) for a, b in zip(fr, to)}
    need = n_line - N - parallel_lines
    # chords span 2..max_span ring positions, like the fixture (case118 spans 2..20)
    while need > 0:
        a = rng.integers(0, N, size=2 * need + 16)
        span = rng.integers(2, max_span + 1, size=a.size)
        for u, sp in zip(a.tolist(), span.tolist()):
            if need == 0:
                break
            v = (u + sp) % N
            key = (min(u, v), max(u, v))
            if u == v or key in seen:
                continue
            seen.add(key)
            fr.append(u)
            to.append(v)
            need -= 1
    for k in range(parallel_lines):
        j = int(rng.integers(0, len(fr)))
        fr.append(to[j] if k % 2 else fr[j])  # reversed orientation every other one
        to.append(fr[j] if k % 2 else to[j])
    L = len(fr)
    r = np.round(rng.uniform(0.005, 0.041, L), 5)
    x = np.round(rng.uniform(0.030, 0.118, L), 5)
    branch = np.zeros((L, 13))
    branch[:, 0] = np.array(fr) + 1
    branch[:, 1] = np.array(to) + 1
    branch[:, 2] = r
    branch[:, 3] = x
    branch[:, 5:8] = 500.0
    branch[:, 10] = 1
    branch[:, 11] = -360.0
    branch[:, 12] = 360.0
    # generators: bus 0 (reference) always carries one
    gbuses = [0] + sorted(rng.choice(np.arange(1, N), size=n_gen - 1, replace=False).tolist())
    if shared_gens:
        gbuses = sorted(gbuses + rng.choice(gbuses, size=shared_gens).tolist())
    G = len(gbuses)
    pmax = np.round(rng.uniform(61.0, 159.0, G), 1)
    gen = np.zeros((G, 10))
    gen[:, 0] = np.array(gbuses) + 1
    gen[:, 1] = np.round(0.56 * pmax, 2)
    gen[:, 3] = np.round(0.6 * pmax, 1)
    gen[:, 4] = -gen[:, 3]
    gen[:, 5] = 1.0
    gen[:, 6] = 100.0
    gen[:, 7] = 1
    gen[:, 8] = pmax
    gencost = np.zeros((G, 7))
    gencost[:, 0] = 2
    gencost[:, 3] = 3
    gencost[:, 4] = np.round(rng.uniform(0.012, 0.05, G), 5)
    gencost[:, 5] = np.round(rng.uniform(8.7, 33.5, G), 3)
    gencost[:, 6] = np.round(rng.uniform(1.7, 60.0, G), 2)
    # buses and loads
    bus = np.zeros((N, 13))
    bus[:, 0] = np.arange(1, N + 1)
    bus[:, 1] = 1
    bus[np.array(gbuses), 1] = 2
    bus[0, 1] = 3
    lb = rng.choice(N, size=n_load, replace=False)
    pd = np.round(rng.uniform(15.0, 55.0, n_load), 2)
    qf = rng.uniform(0.2, 0.45, n_load)
    if load_scale != 1.0:
        pd = np.round(pd * load_scale, 2)
    bus[lb, 2] = pd
    bus[lb, 3] = np.round(pd * qf, 2)
    bus[:, 6] = 1
    bus[:, 7] = 1.0
    bus[:, 9] = 138.0
    bus[:, 10] = 1
    bus[:, 11] = 1.06
    bus[:, 12] = 0.92
    return RawCase(100.0, bus, gen, branch, gencost)


def config_case(name: str, seed: int = 1) -> RawCase:
    return synthetic_case(*CONFIG_SIZES[name], seed=seed)
