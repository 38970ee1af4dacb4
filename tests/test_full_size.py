"""GPU: parity at the bench's full size (synthetic30k x 96 periods), through properties
that do not need a full-size CPU run:

* period locality -- every pattern except ramp is per-period, so the callbacks of the
  96-period problem restricted to a window of 2 periods equal the reference's own
  2-period problem on the same network and load slice (ramp rows inside the window
  included).  g, grad, J and H are compared entry by entry (J/H through their COO
  (row, col) keys mapped into the window problem);
* path identity -- the fused A/M (straight from x) equal set_jacobian(eval_jac(x)) /
  assemble(eval_hess(x)) bit for bit at full size;
* shard identity -- a period shard of the full problem reproduces its rows bit for bit
  (tests/test_shard.py does this exhaustively at small sizes).

Tolerance for values: 1e-12 relative / 1e-14 absolute (CUDA vs glibc sin/cos ulps)."""
import numpy as np
import pytest

from helpers import DELTAS, assert_bitexact, assert_close, interior_point, row_weights, sigmas
from oracle import bindings as B
from paper_2405_14032_b200.abi import GN_IN_FULL
from paper_2405_14032_b200.network import config_case
from paper_2405_14032_b200.opf import CondensedKkt, OpfNlp, load_profile

pytestmark = pytest.mark.gpu

T, T0, TW = 96, 40, 2  # full horizon, window start, window length


@pytest.fixture(scope="module")
def full():
    raw = config_case("synthetic30k")
    net = raw.network()
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 99)
    w = row_weights(nlp.n_cons(), 98, zero_every=11)
    return dict(raw=raw, net=net, scale=scale, nlp=nlp, x=x, w=w)


class _Layout:
    """Row / variable (entity, period) decomposition of the OPF layout (opf.hpp:16-60)."""

    def __init__(self, N, L, G, LT, GR, T):
        self.T = T
        self.voff = np.cumsum([0, G * T, G * T, L * T, L * T, N * T, N * T])
        self.roff = np.cumsum([0, N * T, N * T, L * T, L * T, LT * T, L * T, GR * max(T - 1, 0)])

    def var(self, v):
        b = np.searchsorted(self.voff, v, side="right") - 1
        r = v - self.voff[b]
        return b, r // self.T, r % self.T

    def row(self, r):
        b = np.searchsorted(self.roff, r, side="right") - 1
        q = r - self.roff[b]
        ramp = b == 6
        Tm = max(self.T - 1, 1)
        e = np.where(ramp, q // Tm, q // self.T)
        t = np.where(ramp, q % Tm + 1, q % self.T)  # ramp: the step s (rows pg_s - pg_{s-1})
        return b, e, t

    def var_index(self, b, e, t):
        return self.voff[b] + e * self.T + t

    def row_index(self, b, e, t):
        ramp = b == 6
        return np.where(ramp, self.roff[b] + e * max(self.T - 1, 1) + t - 1,
                        self.roff[b] + e * self.T + t)


def _window(full):
    net, s = full["net"], full["nlp"].sizes
    N, L, G = net.n_bus, net.n_line, net.n_gen
    LT, GR = s.n_thermal, s.n_ramp_gens
    big, small = _Layout(N, L, G, LT, GR, T), _Layout(N, L, G, LT, GR, TW)
    text = full["raw"].to_matpower()
    ref = B.RefModel(text, TW, full["scale"][T0:T0 + TW])
    # window x: every variable block, periods [T0, T0 + TW)
    vb, ve, vt = small.var(np.arange(ref.sizes[0]))
    xw = full["x"][big.var_index(vb, ve, vt + T0)]
    rb, re_, rt = small.row(np.arange(ref.sizes[1]))
    wrow = big.row_index(rb, re_, rt + T0)
    return big, small, ref, xw, wrow


def _coo_window(big, small, rows, cols, vals, nvars_small):
    """Entries of the full COO whose row lies in the window, keyed in the window problem."""
    r = rows.astype(np.int64)
    ramp = r >= big.roff[6]
    t = np.where(ramp, (r - big.roff[6]) % max(T - 1, 1) + 1, r % T)
    keep = np.flatnonzero((t >= T0) & (t < T0 + TW) & (~ramp | (t > T0)))  # ramp: steps T0+1..
    rb, re_, rt = big.row(r[keep])
    rt = rt - T0
    cb, ce, ct = big.var(cols[keep].astype(np.int64))
    assert np.all((ct >= T0) & (ct < T0 + TW)), "a window row references a period outside it"
    vals = vals[keep]
    key = small.row_index(rb, re_, rt) * nvars_small + small.var_index(cb, ce, ct - T0)
    return key, vals


def _summed(key, vals):
    o = np.argsort(key, kind="stable")
    key, vals = key[o], vals[o]
    u, start = np.unique(key, return_index=True)
    return u, np.add.reduceat(vals, start) if len(vals) else vals


def test_period_locality_callbacks(full):
    nlp = full["nlp"]
    big, small, ref, xw, wrow = _window(full)
    ok, g = nlp.eval_g(full["x"])
    okr, gr, _ = ref.eval_g(xw)
    assert ok and okr
    assert_close(g[wrow], gr, what="g window")
    ok, grad = nlp.eval_grad(full["x"])
    okr, gradr, _ = ref.eval_grad(xw)
    vb, ve, vt = small.var(np.arange(ref.sizes[0]))
    assert_bitexact(grad[big.var_index(vb, ve, vt + T0)], gradr, "grad window")
    jr, jc = nlp.jac_structure()
    hr, hc = nlp.hess_structure()
    rjr, rjc, rhr, rhc = ref.structure()
    nvs = ref.sizes[0]
    ok, J = nlp.eval_jac(full["x"])
    okr, Jr, _ = ref.eval_jac(xw)
    assert ok and okr
    k, v = _coo_window(big, small, jr, jc, J, nvs)
    u, s_ = _summed(k, v)
    ur, sr = _summed(rjr.astype(np.int64) * nvs + rjc, Jr)
    assert np.array_equal(u, ur), "J window pattern"
    assert_close(s_, sr, what="J window")
    wv = full["w"]
    ok, H = nlp.eval_hess(full["x"], wv, 0.8)
    okr, Hr, _ = ref.eval_hess(xw, wv[wrow], 0.8)
    assert ok and okr
    # H entries whose two variables both lie in the window (every variable block's offset
    # is a multiple of T, so the period is the index mod T).  Entries across the window
    # edge come only from ramp steps outside it; ramp Hessians are zero, so the summed
    # values of the kept keys are the window problem's.
    keep = np.flatnonzero(((hr % T) >= T0) & ((hr % T) < T0 + TW) &
                          ((hc % T) >= T0) & ((hc % T) < T0 + TW))
    rb, re_, rt = big.var(hr[keep].astype(np.int64))
    cb, ce, ct = big.var(hc[keep].astype(np.int64))
    key = small.var_index(rb, re_, rt - T0) * nvs + small.var_index(cb, ce, ct - T0)
    u, s_ = _summed(key, H[keep])
    ur, sr = _summed(rhr.astype(np.int64) * nvs + rhc, Hr)
    assert np.array_equal(u, ur), "H window pattern"
    assert_close(s_, sr, what="H window")


def test_fused_equals_contract_full_size(full):
    nlp = full["nlp"]
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    assert K.fused_ready == 1
    sx, ss = sigmas(nlp.sizes.n_free, nlp.n_cons(), 97)
    ok, jv = nlp.eval_jac(full["x"])
    ok2, hv = nlp.eval_hess(full["x"], full["w"], 1.0)
    assert ok and ok2
    for dw, dc in DELTAS:
        K.set_jacobian(jv, mem=GN_IN_FULL)
        K.assemble(hv, sx, ss, dw, dc, mem=GN_IN_FULL)
        a_ref, m_ref = K.values()
        K.update_x(full["x"], full["w"], 1.0, sx, ss, dw, dc)
        a, m = K.values()
        assert_bitexact(a, a_ref, f"A full size dw={dw}")
        assert_bitexact(m, m_ref, f"M full size dw={dw}")
