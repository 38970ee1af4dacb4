"""Shared test inputs and comparators (SURVEY.md §8(d) input recipe)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# Value tolerance from BASELINE.json north_star: 1e-12 relative, 1e-14 absolute floor.
REL, ABS = 1e-12, 1e-14


def interior_point(xl, xu, xs, seed=1234):
    """acceptance.cpp:274-284 recipe (numpy stream): two-sided boxes get
    lo + (0.15 + 0.7u)(hi - lo), free variables start + 0.2(u - 0.5), fixed = lo."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(size=len(xl))
    both = np.isfinite(xl) & np.isfinite(xu)
    with np.errstate(invalid="ignore"):
        x = np.where(both, xl + (0.15 + 0.7 * u) * (xu - xl), xs + 0.2 * (u - 0.5))
    return np.where(xl == xu, xl, x)


def row_weights(m, seed=7, zero_every=0):
    w = -np.random.default_rng(seed).uniform(-1.0, 1.0, m)  # w = -y, y ~ U(-1,1)
    if zero_every:
        w[::zero_every] = 0.0
        w[1::2 * zero_every] = -0.0
    return w


def sigmas(n, m, seed=11):
    rng = np.random.default_rng(seed)
    return 10.0 ** rng.uniform(-2, 2, n), 10.0 ** rng.uniform(-2, 2, m)


DELTAS = [(0.0, 0.0), (1e-4, 1e-8 * 0.1 ** 0.25)]


def assert_close(got, ref, rel=REL, abs_=ABS, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    if got.size == 0:
        return
    err = np.abs(got - ref)
    tol = np.maximum(rel * np.abs(ref), abs_)
    bad = ~(err <= tol)
    if bad.any():
        i = int(np.argmax(np.where(bad, err / tol, 0)))
        raise AssertionError(f"{what}: {int(bad.sum())} of {got.size} outside tolerance; "
                             f"worst at {i}: got {got[i]!r} ref {ref[i]!r}")


def assert_bitexact(got, ref, what=""):
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    if got.dtype.kind == "f":
        bad = ~((got == ref) | (np.isnan(got) & np.isnan(ref)))
    else:
        bad = got != ref
    if bad.any():
        i = int(np.argmax(bad))
        raise AssertionError(f"{what}: {int(bad.sum())} of {got.size} differ; first at {i}: "
                             f"got {got[i]!r} ref {ref[i]!r}")


def golden_network(case: str):
    """Reference-parsed network fixture (tests/golden/networks.npz)."""
    from paper_2405_14032_b200.network import Network
    z = np.load(GOLDEN / "networks.npz")
    kw = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(case + "/")}
    base = float(kw.pop("base_mva"))
    ref = int(kw.pop("reference_bus"))
    return Network(base_mva=base, reference_bus=ref, **kw)


def golden_eval(name: str):
    return np.load(GOLDEN / f"eval_{name}.npz")


def golden_meta():
    return json.loads((GOLDEN / "meta.json").read_text())
