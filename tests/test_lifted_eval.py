"""GPU: the lifted evaluations (gn_lifted_eval_*, LiftedProblem::eval_* at lifted.hpp:
128-159 in one library call each) against the reference's own lifted values in the golden
fixtures, and against the library's full-space call + gather.  These back the shim
LiftedProblem (include/gridnlp_b200/shim/gridnlp/ipm/lifted.hpp) the drop-in uses."""
import numpy as np
import pytest

from helpers import assert_bitexact, assert_close, golden_eval, golden_meta, golden_network
from paper_2405_14032_b200.abi import GN_ERR_INVALID, GN_ERR_UNSUPPORTED, GN_MEM_DEVICE
from paper_2405_14032_b200.opf import GridError, OpfNlp

pytestmark = pytest.mark.gpu
FIXTURES = list(golden_meta()["fixtures"])


def _lifted(fx):
    meta = golden_meta()["fixtures"][fx]
    z = golden_eval(fx)
    net = golden_network(meta["case"])
    nlp = OpfNlp(net, meta["periods"], z["scale"]).lift(1e-4)
    return nlp, z, net, meta


@pytest.mark.parametrize("fx", FIXTURES)
@pytest.mark.parametrize("mem", ["host", "device"])
def test_lifted_eval_matches_reference(gpu, fx, mem):
    import torch
    nlp, z, _, _ = _lifted(fx)
    f2f = z["l_free_to_full"]
    x, w, ow = z["x"], z["w"], float(z["ow"])
    xf = x[f2f]
    if mem == "host":
        call = lambda which, **kw: nlp.lifted_eval(which, xf, **kw)[1]  # noqa: E731
        ok_f, f = nlp.lifted_eval("f", xf)
        assert ok_f
        f = float(f[0])
    else:
        dev = torch.device("cuda", 0)
        dxf = torch.from_numpy(xf).to(dev)
        dw = torch.from_numpy(w).to(dev)
        s = nlp.sizes
        sizes = {"grad": s.n_free, "g": s.n_cons, "jac": s.jac_nnz_lifted,
                 "hess": s.hess_nnz_lifted, "f": 1}

        def call(which, w=None, ow=1.0):
            out = torch.full((sizes[which],), np.nan, dtype=torch.float64, device=dev)
            ok, _ = nlp.lifted_eval(which, dxf, w=dw if w is not None else None, ow=ow, out=out,
                                    mem=GN_MEM_DEVICE)
            assert ok
            return out.cpu().numpy()
        f = float(call("f")[0])
    assert_close([f], [float(z["f"])], what="lifted f")
    assert_bitexact(call("grad"), z["grad"][f2f], "lifted grad")
    assert_close(call("g"), z["g"], what="lifted g")
    jl = call("jac")
    hl = call("hess", w=w, ow=ow)
    assert_close(jl, z["jac_l"], what="lifted jac")
    assert_close(hl, z["hess_l"], what="lifted hess")
    # the same values the full-space call + the library's gather produce, bit for bit
    ok, jac = nlp.eval_jac(x)
    ok2, hess = nlp.eval_hess(x, w, ow)
    assert ok and ok2
    assert_bitexact(jl, nlp.lifted_gather("jac", jac), "lifted jac == gather(full)")
    assert_bitexact(hl, nlp.lifted_gather("hess", hess), "lifted hess == gather(full)")
    if mem == "host":
        ok, (fg_f, fg_g) = nlp.lifted_eval("fg", xf)
        assert ok
        assert fg_f == f
        assert_bitexact(fg_g, call("g"), "lifted fg: g")


def test_lifted_eval_pins_fixed_entries(gpu):
    """The staging writes only the free entries; fixed ones keep their pinned values
    (lifted.hpp:35-45): whatever the caller's full point held there does not matter."""
    nlp, z, _, meta = _lifted("case118_T4")
    f2f = z["l_free_to_full"]
    x = z["x"].copy()
    fixed = np.setdiff1d(np.arange(len(x)), f2f)
    assert len(fixed) > 0  # th_ref at least
    x_pinned = x.copy()
    x_pinned[fixed] = z["xl"][fixed]
    ok, g_ref = nlp.eval_g(x_pinned)
    assert ok
    ok, g = nlp.lifted_eval("g", x[f2f])
    assert ok
    assert_bitexact(g, g_ref, "lifted g at the pinned point")


def test_lifted_eval_failure_report(gpu):
    """A non-finite free variable fails the lifted call exactly like the full call at the
    corresponding full index: same (pattern, record), ok False, status cleared after."""
    nlp, z, _, _ = _lifted("synth_T3")
    f2f = z["l_free_to_full"]
    xf = z["x"][f2f].copy()
    for k in (len(xf) // 2, len(xf) - 3, 5):
        bad = xf.copy()
        bad[k] = np.nan
        full = z["x"].copy()
        full[f2f[k]] = np.nan
        for which, kw, full_call in (
                ("g", {}, lambda: nlp.eval_g(full)),
                ("jac", {}, lambda: nlp.eval_jac(full)),
                ("hess", {"w": z["w"], "ow": 0.7}, lambda: nlp.eval_hess(full, z["w"], 0.7))):
            okf, _ = full_call()
            err_full = nlp.last_error if not okf else None
            ok, _ = nlp.lifted_eval(which, bad, **kw)
            assert ok == okf, (which, k)
            if not ok:
                assert nlp.last_error == err_full, (which, k)
    ok, _ = nlp.lifted_eval("g", xf)
    assert ok


def test_lifted_eval_needs_lift(gpu):
    from paper_2405_14032_b200.opf import _f64
    meta = golden_meta()["fixtures"]["case9_T2"]
    z = golden_eval("case9_T2")
    nlp = OpfNlp(golden_network(meta["case"]), 2, z["scale"])
    out = np.empty(len(z["g"]))
    assert nlp.lib.gn_lifted_eval_g(nlp.h, _f64(z["x"]), _f64(out), 0, None) == GN_ERR_INVALID


def test_lifted_eval_rejects_period_shard(gpu):
    from paper_2405_14032_b200.network import synthetic_case
    from paper_2405_14032_b200.opf import load_profile
    net = synthetic_case(20, 30, 6, 12, seed=3).network()
    T_total, T, t0 = 6, 3, 3
    scale = load_profile(net.n_load, T_total)
    nlp = OpfNlp(net, T, scale[t0:t0 + T], shard=(T_total, t0)).lift(1e-4)
    with pytest.raises(GridError) as e:
        nlp.lifted_eval("g", np.zeros(nlp.sizes.n_free))
    assert e.value.code == GN_ERR_UNSUPPORTED


@pytest.mark.parametrize("seed", range(4))
def test_lifted_eval_randomised_fixed_variables(gpu, seed):
    """Random networks with fixed generators (pmin == pmax > 0) and fixed voltages, so the
    pinned values enter g, J and H: the lifted calls on the free-variable vector equal the
    bit-exact C restatement's full-space evaluation at the pinned point, gathered by its
    own lifted picks (grad bit-exact, the rest within the 1e-12 bar)."""
    from oracle import bindings as B
    from helpers import interior_point, row_weights
    from paper_2405_14032_b200.network import synthetic_case
    from paper_2405_14032_b200.opf import load_profile
    rng = np.random.default_rng(500 + seed)
    N = int(rng.integers(20, 150))
    raw = synthetic_case(N, N + int(rng.integers(N // 3, N)), int(rng.integers(4, 20)),
                         int(rng.integers(N // 3, N)), seed=int(rng.integers(1, 10_000)),
                         parallel_lines=int(rng.integers(0, 3)))
    net = raw.network()
    for g in rng.choice(net.n_gen, size=min(3, net.n_gen), replace=False):
        net.gen_pmin[g] = net.gen_pmax[g] = max(net.gen_pmax[g], 0.3)
    for b in rng.choice(net.n_bus, size=3, replace=False):
        if b != net.reference_bus:
            net.bus_vmin[b] = net.bus_vmax[b] = 1.02
    T = int(rng.integers(1, 40))
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale).lift(1e-4)
    orc = B.OracleModel(net, T, scale)
    lo = orc.lift(1e-4)
    ours = nlp.lifted_structure()
    assert_bitexact(ours["free_to_full"], lo["free_to_full"], "free_to_full")
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, seed)
    fixed = xl == xu
    assert fixed.sum() > 3 * T  # generators and voltages pinned, not only th_ref
    x[fixed] = xl[fixed]  # the pinned point
    xf = x[lo["free_to_full"]]
    w = row_weights(nlp.sizes.n_cons, seed + 3)
    ow = float(rng.uniform(0.2, 2.0))
    ok, g = nlp.lifted_eval("g", xf)
    okg, go, _ = orc.eval_g(x)
    assert ok and okg
    assert_close(g, go, what="lifted g")
    ok, gr = nlp.lifted_eval("grad", xf)
    okg, gro, _ = orc.eval_grad(x)
    assert ok and okg
    assert_bitexact(gr, gro[lo["free_to_full"]], "lifted grad")
    ok, jl = nlp.lifted_eval("jac", xf)
    okj, jo, _ = orc.eval_jac(x)
    assert ok and okj
    assert_close(jl, jo[lo["jac_pick"]], what="lifted jac")
    ok, hl = nlp.lifted_eval("hess", xf, w=w, ow=ow)
    okh, ho, _ = orc.eval_hess(x, w, ow)
    assert ok and okh
    assert_close(hl, ho[lo["hess_pick"]], what="lifted hess")
