"""GPU: device-resident IPM vector operations against the compiled
reference (oracle/_ref: ipm/iterate.hpp, CondensedKkt::solve's vector parts).

Element-wise results and the sparse products (J^T y and J x in COO order, A^T v in
CSR row order, A v per row) must be bit-identical; fraction_to_boundary is a min and
must be exact; whole-vector sums (barrier value and slope, constraint violation, the
kkt_error scalings) use a fixed reduction tree and must agree to 1e-12 relative."""
import numpy as np
import pytest

from oracle import bindings as B
from paper_2405_14032_b200.network import synthetic_case
from paper_2405_14032_b200.opf import CondensedKkt, Ipm, OpfNlp

pytestmark = pytest.mark.gpu

REL = 1e-12


def _rel(a, b):
    return abs(a - b) <= REL * max(1.0, abs(b))


@pytest.fixture(scope="module", params=[(300, 470, 60, 250, 4, 0), (120, 190, 30, 100, 3, 4)])
def setup(request):
    import torch
    N, L, G, D, T, par = request.param
    raw = synthetic_case(N, L, G, D, seed=11 + par, parallel_lines=par, shared_gens=par)
    text = raw.to_matpower()
    net = raw.network()
    scale = B.ref_load_profile(text, T)
    ref = B.RefModel(text, T, scale)
    ref.lift(1e-4)
    ref.kkt_create()
    nlp = OpfNlp(net, T, scale)
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    bounds = ref.lifted_bounds()
    n, m = ref.lifted_sizes[0], ref.lifted_sizes[1]
    assert (n, m) == (nlp.sizes.n_free, nlp.sizes.n_cons)
    rng = np.random.default_rng(5)
    xl, xu, sl, su = bounds
    # interior iterate, multipliers on present bounds only (Iterate convention)
    def interior(lo, hi, k):
        base = np.where(np.isfinite(lo), lo, np.where(np.isfinite(hi), hi - 2.0, 0.0))
        width = np.where(np.isfinite(lo) & np.isfinite(hi), hi - lo, 2.0)
        return base + (0.1 + 0.8 * rng.random(k)) * width
    x, s = interior(xl, xu, n), interior(sl, su, m)
    y = rng.uniform(-1, 1, m)
    zlx = np.where(np.isfinite(xl), rng.uniform(0.01, 2, n), 0.0)
    zux = np.where(np.isfinite(xu), rng.uniform(0.01, 2, n), 0.0)
    zls = np.where(np.isfinite(sl), rng.uniform(0.01, 2, m), 0.0)
    zus = np.where(np.isfinite(su), rng.uniform(0.01, 2, m), 0.0)
    it = [x, s, y, zlx, zux, zls, zus]
    nj = ref.lifted_sizes[2]
    jv = rng.uniform(-3, 3, nj)
    grad = rng.uniform(-5, 5, n)
    g = rng.uniform(-1, 1, m)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ipm = Ipm(K, *bounds)
    return dict(ref=ref, K=K, ipm=ipm, it=it, jv=jv, grad=grad, g=g, t=t, n=n, m=m,
                bounds=bounds, rng=rng, torch=torch)


def _cpu(ts):
    return [v.cpu().numpy() for v in ts]


def test_jacobian_products(setup):
    S = setup
    t, ipm, ref = S["t"], S["ipm"], S["ref"]
    y = S["rng"].uniform(-1, 1, S["m"])
    xv = S["rng"].uniform(-1, 1, S["n"])
    out_n = S["torch"].empty(S["n"], dtype=S["torch"].float64, device="cuda")
    out_m = S["torch"].empty(S["m"], dtype=S["torch"].float64, device="cuda")
    ipm.jac_transpose_multiply(t(S["jv"]), t(y), out_n)
    ipm.jac_multiply(t(S["jv"]), t(xv), out_m)
    assert np.array_equal(out_n.cpu().numpy(), ref.ipm_jac_t(S["jv"], y))
    assert np.array_equal(out_m.cpu().numpy(), ref.ipm_jac(S["jv"], xv))


def _residuals(S, mu):
    torch, t = S["torch"], S["t"]
    nm = [S["n"], S["m"], S["m"], S["n"], S["n"], S["m"], S["m"]]
    r = [torch.empty(k, dtype=torch.float64, device="cuda") for k in nm]
    S["ipm"].residuals([t(a) for a in S["it"]], t(S["grad"]), t(S["g"]), t(S["jv"]), mu, r)
    return r


@pytest.mark.parametrize("mu", [0.0, 0.1])
def test_residuals_condensation_kkt_error(setup, mu):
    S = setup
    ref, t, torch = S["ref"], S["t"], S["torch"]
    r = _residuals(S, mu)
    rr = ref.ipm_residuals(S["bounds"], S["it"], S["grad"], S["g"], S["jv"], mu)
    for a, b, name in zip(_cpu(r), rr, ["px", "ps", "py", "pzlx", "pzux", "pzls", "pzus"]):
        assert np.array_equal(a, b), name
    n, m = S["n"], S["m"]
    out = [torch.empty(k, dtype=torch.float64, device="cuda") for k in (n, m, n, m)]
    S["ipm"].bound_condensation([t(a) for a in S["it"]], r, *out)
    for a, b, name in zip(_cpu(out), ref.ipm_condense(S["bounds"], S["it"], rr),
                          ["sigma_x", "sigma_s", "qx", "qs"]):
        assert np.array_equal(a, b), name
    e = S["ipm"].kkt_error([t(a) for a in S["it"]], r, mu)
    er = ref.ipm_kkt_error(S["bounds"], S["it"], rr, mu)
    for a, b, name in zip(e, er, ["stat", "feas", "comp"]):
        assert _rel(a, b), (name, a, b)
    assert e[1] == er[1]  # feas is a max: exact


def test_steps_boundary_barrier(setup):
    S = setup
    ref, t, torch, rng = S["ref"], S["t"], S["torch"], S["rng"]
    n, m = S["n"], S["m"]
    mu = 0.05
    r = _residuals(S, mu)
    rr = ref.ipm_residuals(S["bounds"], S["it"], S["grad"], S["g"], S["jv"], mu)
    dx, ds, dy = rng.uniform(-1, 1, n), rng.uniform(-1, 1, m), rng.uniform(-1, 1, m)
    dd = [t(dx), t(ds), t(dy)] + [torch.empty(k, dtype=torch.float64, device="cuda")
                                  for k in (n, n, m, m)]
    S["ipm"].recover_bound_steps([t(a) for a in S["it"]], r, dd)
    dz_ref = ref.ipm_recover(S["bounds"], S["it"], rr, [dx, ds, dy] + [np.zeros(k) for k in (n, n, m, m)])
    for a, b, name in zip(_cpu(dd[3:]), dz_ref, ["dzlx", "dzux", "dzls", "dzus"]):
        assert np.array_equal(a, b), name
    d_np = [dx, ds, dy] + dz_ref
    for tau in (0.99, 0.995):
        a = S["ipm"].fraction_to_boundary([t(v) for v in S["it"]], dd, tau)
        assert a == list(ref.ipm_ftb(S["bounds"], S["it"], d_np, tau))
    f = 123.456
    bv = S["ipm"].barrier_value(f, t(S["it"][0]), t(S["it"][1]), mu)[0]
    assert _rel(bv, ref.ipm_barrier(S["bounds"], f, S["it"][0], S["it"][1], mu))
    sl = S["ipm"].barrier_slope(t(S["grad"]), [t(v) for v in S["it"]], dd, mu)[0]
    assert _rel(sl, ref.ipm_slope(S["bounds"], S["grad"], S["it"], d_np, mu))
    cv = S["ipm"].constraint_violation(t(S["g"]), t(S["it"][1]))[0]
    assert _rel(cv, ref.ipm_violation(S["g"], S["it"][1]))


@pytest.mark.parametrize("dw,dc", [(0.0, 0.0), (1e-4, 1e-8 * 0.1 ** 0.25)])
def test_condensed_solve_vector_parts(setup, dw, dc):
    S = setup
    ref, t, torch, rng, K = S["ref"], S["t"], S["torch"], S["rng"], S["K"]
    n, m = S["n"], S["m"]
    ref.kkt_set_jacobian(S["jv"])
    K.set_jacobian(t(S["jv"]), mem=1)  # GN_MEM_DEVICE, lifted J values
    qx, qs, qy = rng.uniform(-1, 1, n), rng.uniform(-1, 1, m), rng.uniform(-1, 1, m)
    ss = 10.0 ** rng.uniform(-2, 2, m)
    dx = rng.uniform(-1, 1, n)
    rhs_ref, ds_ref, dy_ref = ref.kkt_solve_parts(qx, qs, qy, ss, dw, dc, dx)
    rhs = torch.empty(n, dtype=torch.float64, device="cuda")
    ds = torch.empty(m, dtype=torch.float64, device="cuda")
    dy = torch.empty(m, dtype=torch.float64, device="cuda")
    S["ipm"].solve_rhs(t(qx), t(qs), t(qy), t(ss), dw, dc, rhs)
    S["ipm"].solve_finish(t(dx), t(qs), t(qy), t(ss), dw, dc, ds, dy)
    assert np.array_equal(rhs.cpu().numpy(), rhs_ref)
    assert np.array_equal(ds.cpu().numpy(), ds_ref)
    assert np.array_equal(dy.cpu().numpy(), dy_ref)
