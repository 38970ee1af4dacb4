"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
fixtures and the bit-exact oracle.

Bar (BASELINE.json north_star): structures and scatter maps bit-exact; values
within 1e-12 relative with a 1e-14 absolute floor (helpers.REL/ABS); sums with
no transcendental (balance rows, gradient, A, M given equal inputs) bit-exact.
"""
import os

import numpy as np
import pytest

from helpers import (DELTAS, assert_bitexact, assert_close, golden_eval, golden_meta,
                     golden_network, interior_point, row_weights, sigmas)
from oracle import bindings as B
from paper_2405_14032_b200.abi import GN_IN_FULL, GN_MEM_DEVICE
from paper_2405_14032_b200.network import synthetic_case
from paper_2405_14032_b200.opf import CondensedKkt, GridError, OpfNlp, compress_to_csc

pytestmark = pytest.mark.gpu
FIXTURES = list(golden_meta()["fixtures"])


def _nlp(fx):
    meta = golden_meta()["fixtures"][fx]
    z = golden_eval(fx)
    net = golden_network(meta["case"])
    return OpfNlp(net, meta["periods"], z["scale"]), z, meta, net


def _bal_rows(meta, net):
    T = meta["periods"]
    return np.arange(2 * net.n_bus * T)  # balance_p then balance_q blocks


@pytest.mark.parametrize("fx", FIXTURES)
def test_structure_and_bounds_bitexact(gpu, fx):
    nlp, z, meta, _ = _nlp(fx)
    s = nlp.sizes
    assert [s.n_vars, s.n_cons, s.jac_nnz, s.hess_nnz, s.n_thermal, s.n_ramp_gens] == meta["sizes"]
    for got, key in zip(nlp.bounds(), ("xl", "xu", "xs", "rl", "ru")):
        assert_bitexact(got, z[key], key)
    jr, jc = nlp.jac_structure()
    hr, hc = nlp.hess_structure()
    assert_bitexact(jr, z["jr"], "jac_rows")
    assert_bitexact(jc, z["jc"], "jac_cols")
    assert_bitexact(hr, z["hr"], "hess_rows")
    assert_bitexact(hc, z["hc"], "hess_cols")


@pytest.mark.parametrize("fx", FIXTURES)
def test_callbacks_match_reference(gpu, fx):
    nlp, z, meta, net = _nlp(fx)
    x, w, ow = z["x"], z["w"], float(z["ow"])
    ok, f = nlp.eval_f(x)
    assert ok
    assert_close([f], [float(z["f"])], what="f")
    ok, grad = nlp.eval_grad(x)
    assert ok
    assert_bitexact(grad, z["grad"], "grad")  # c1 + (2 c2) pg, same rounding
    ok, g = nlp.eval_g(x)
    assert ok
    assert_close(g, z["g"], what="g")
    bal = _bal_rows(meta, net)
    assert_bitexact(g[bal], z["g"][bal], "balance rows (canonical order)")
    ok, jac = nlp.eval_jac(x)
    assert ok
    assert_close(jac, z["jac"], what="jac")
    ok, hess = nlp.eval_hess(x, w, ow)
    assert ok
    assert_close(hess, z["hess"], what="hess")
    # w == 0 (and -0.0) rows: every slot of those records is +0.0 (pattern_model.hpp:409-412)
    assert np.all(hess[z["hess"] == 0.0] == 0.0)


@pytest.mark.parametrize("fx", FIXTURES)
def test_lifted_filter_bitexact(gpu, fx):
    nlp, z, meta, net = _nlp(fx)
    nlp.lift(1e-4)
    s = nlp.sizes
    assert [s.n_free, s.n_cons, s.jac_nnz_lifted, s.hess_nnz_lifted] == meta["lifted"]
    L = nlp.lifted_structure()
    for k in ("free_to_full", "jac_rows", "jac_cols", "hess_rows", "hess_cols", "s_lower",
              "s_upper"):
        assert_bitexact(L[k], z["l_" + k], k)
    orc = B.OracleModel(net, meta["periods"], z["scale"])
    lo = orc.lift(1e-4)
    assert_bitexact(L["jac_pick"], lo["jac_pick"], "jac_pick")
    assert_bitexact(L["hess_pick"], lo["hess_pick"], "hess_pick")


@pytest.mark.parametrize("fx", FIXTURES)
@pytest.mark.parametrize("mode", ["lifted-host", "full-host", "generic", "published"])
def test_kkt_structure_slots_and_values_bitexact(gpu, fx, mode):
    """generic: gn_kkt_create on the lifted COO arrays (the reference IpmSolver's call,
    solver.hpp:139-141) -> contributor-list kernels; published: the same call after
    gn_ctx_publish -> recognised as the OPF problem, specialised kernels on lifted inputs."""
    nlp, z, meta, net = _nlp(fx)
    if mode == "published":
        nlp.publish()  # lifts the problem
    else:
        nlp.lift(1e-4)
    if mode in ("generic", "published"):
        K = CondensedKkt(meta["lifted"][0], meta["sizes"][1], z["l_jac_rows"], z["l_jac_cols"],
                         z["l_hess_rows"], z["l_hess_cols"])
        assert K.opf_ready == (1 if mode == "published" else 0)
    else:
        K = CondensedKkt(nlp=nlp)
    assert [K.dim, K.a_nnz, K.m_nnz] == meta["kkt"]
    for got, key in zip(K.structure(), ("rowptr", "colidx", "colptr", "rowidx")):
        assert_bitexact(got, z[key], key)
    orc = B.OracleModel(net, meta["periods"], z["scale"])
    orc.lift(1e-4)
    OK = orc.kkt()
    for got, ref, name in zip(K.slots(), OK.slots(), ("jac", "hess", "pair", "diag")):
        assert_bitexact(got, ref, name + "_slots")
    if mode == "full-host":
        K.set_jacobian(z["jac"], mem=GN_IN_FULL)
    else:
        K.set_jacobian(z["jac_l"])
    for i, (dw, dc) in enumerate(DELTAS):
        if mode == "full-host":
            K.assemble(z["hess"], z["sx"], z["ss"], dw, dc, mem=GN_IN_FULL)
        else:
            K.assemble(z["hess_l"], z["sx"], z["ss"], dw, dc)
        a, m = K.values()
        assert_bitexact(a, z["avals"], "A values")
        assert_bitexact(m, z[f"mvals{i}"], f"M values delta#{i}")


def test_device_resident_path_matches_host(gpu):
    import torch
    nlp, z, meta, net = _nlp("case118_T4")
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    x, w = t(z["x"]), t(z["w"])
    s = nlp.sizes
    f = torch.zeros(1, dtype=torch.float64, device=dev)
    grad = torch.empty(s.n_vars, dtype=torch.float64, device=dev)
    g = torch.empty(s.n_cons, dtype=torch.float64, device=dev)
    J = torch.empty(s.jac_nnz, dtype=torch.float64, device=dev)
    H = torch.empty(s.hess_nnz, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    assert nlp.eval_device("f", x, f)
    assert nlp.eval_device("grad", x, grad)
    assert nlp.eval_device("g", x, g)
    assert nlp.eval_device("jac", x, J)
    assert nlp.eval_device("hess", x, H, w=w, ow=float(z["ow"]))
    for got, name in [(grad, "grad"), (g, "g"), (J, "jac"), (H, "hess")]:
        ok, ref = getattr(nlp, "eval_" + name)(z["x"]) if name != "hess" else \
            nlp.eval_hess(z["x"], z["w"], float(z["ow"]))
        assert_bitexact(got.cpu().numpy(), ref, name)
    sx, ss = t(z["sx"]), t(z["ss"])
    K.set_jacobian(J, mem=GN_MEM_DEVICE | GN_IN_FULL)
    K.assemble(H, sx, ss, 0.0, 0.0, mem=GN_MEM_DEVICE | GN_IN_FULL)
    a, m = K.values()
    assert_close(m, z["mvals0"], what="M from device-resident callbacks")


def test_async_status_and_failure_report(gpu):
    nlp, z, meta, net = _nlp("synth_T3")
    orc = B.OracleModel(net, meta["periods"], z["scale"])
    x = z["x"].copy()
    n = meta["sizes"][0]
    for idx in (n // 2, n - 3, 5):  # a flow, an angle, a generator
        xb = x.copy()
        xb[idx] = np.nan
        for name, args in [("eval_f", (xb,)), ("eval_grad", (xb,)), ("eval_g", (xb,)),
                           ("eval_jac", (xb,)), ("eval_hess", (xb, z["w"], 0.7))]:
            okg, _ = getattr(nlp, name)(*args)
            oko, _, fail = getattr(orc, name)(*args)
            assert okg == oko, (name, idx)
            if not okg:
                assert nlp.last_error == fail, (name, idx, nlp.last_error, fail)
    ok, _ = nlp.eval_g(x)
    assert ok  # status cleared after a failure


@pytest.mark.parametrize("T", [1, 4])
def test_self_loop_lines_match_reference(gpu, T):
    """Self-loop lines (from == to; the reference parser accepts them, matpower.hpp:245-246):
    their records name one variable in two fields, so J carries duplicate coordinates and the
    Hessian's mirrored (v_t, v_f) / (th_t, th_f) entries fold onto one diagonal slot whose value
    doubles (double_slots, pattern_model.hpp:193-197, 433).  Structures, bounds and the lifted
    maps bit-exact, callbacks within 1e-12, balance rows bit-exact (to-then-from), and the KKT
    -- the generic assembly, since the topology kernels need two terminals -- bit-exact against
    the reference's CondensedKkt fed the same values; the fused path is unavailable (loud)."""
    from paper_2405_14032_b200.abi import GN_ERR_UNSUPPORTED
    raw = synthetic_case(40, 64, 10, 30, seed=12, parallel_lines=2)
    raw.branch[3, 1] = raw.branch[3, 0]
    raw.branch[20, 0] = raw.branch[20, 1]
    text = raw.to_matpower()
    scale = B.ref_load_profile(text, T)
    ref = B.RefModel(text, T, scale)
    net = B.ref_parse_matpower(text)
    nlp = OpfNlp(net, T, scale)
    s = nlp.sizes
    assert [s.n_vars, s.n_cons, s.jac_nnz, s.hess_nnz] == ref.sizes[:4]
    for got, want, k in zip(nlp.bounds(), ref.bounds(), ("xl", "xu", "xs", "rl", "ru")):
        assert_bitexact(got, want, k)
    rjr, rjc, rhr, rhc = ref.structure()
    assert_bitexact(nlp.jac_structure()[0], rjr, "jr")
    assert_bitexact(nlp.jac_structure()[1], rjc, "jc")
    assert_bitexact(nlp.hess_structure()[0], rhr, "hr")
    assert_bitexact(nlp.hess_structure()[1], rhc, "hc")
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 7)
    w = row_weights(s.n_cons, 8, zero_every=5)
    for k in ("grad", "g", "jac"):
        ok, v = getattr(nlp, "eval_" + k)(x)
        okr, vr, _ = getattr(ref, "eval_" + k)(x)
        assert ok and okr
        assert_close(v, vr, what=k)
    bal = np.arange(2 * net.n_bus * T)
    assert_bitexact(nlp.eval_g(x)[1][bal], ref.eval_g(x)[1][bal], "balance rows")
    ok, H = nlp.eval_hess(x, w, 0.8)
    okr, Hr, _ = ref.eval_hess(x, w, 0.8)
    assert ok and okr
    assert_close(H, Hr, what="hess (double_slots)")
    nlp.lift(1e-4)
    lift = ref.lift(1e-4)
    L = nlp.lifted_structure()
    for k in ("free_to_full", "jac_rows", "jac_cols", "hess_rows", "hess_cols"):
        assert_bitexact(L[k], lift[k], k)
    K = CondensedKkt(nlp=nlp)
    assert K.opf_ready == 0 and K.fused_ready == 0
    ref.kkt_create()
    for got, want, k in zip(K.structure(), ref.kkt_structure(), ("rowptr", "colidx", "colptr", "rowidx")):
        assert_bitexact(got, want, k)
    okj, jr_ = ref.eval_jac(x)[:2]
    okh, hr_ = ref.eval_hess(x, w, 0.8)[:2]
    jl, hl = jr_[L["jac_pick"]], hr_[L["hess_pick"]]
    sx, ss = sigmas(nlp.sizes.n_free, s.n_cons, 9)
    ref.kkt_set_jacobian(jl)
    K.set_jacobian(jl)
    for dw, dc in DELTAS:
        ref.kkt_assemble(hl, sx, ss, dw, dc)
        K.assemble(hl, sx, ss, dw, dc)
        a, m = K.values()
        ar, mr = ref.kkt_values()
        assert_bitexact(a, ar, "A")
        assert_bitexact(m, mr, f"M dw={dw}")
    with pytest.raises(GridError) as e:
        K.update_x(x, w, 1.0, sx, ss, 0.0, 0.0)
    assert e.value.code == GN_ERR_UNSUPPORTED
    K.close()


def test_compress_to_csc_known_answer_gpu(gpu):
    cp, ri, sm = compress_to_csc(3, 2, [0, 1, 0, 2], [0, 0, 0, 1])
    assert cp.tolist() == [0, 2, 3] and ri.tolist() == [0, 1, 2] and sm.tolist() == [0, 1, 0, 2]
    with pytest.raises(GridError):
        compress_to_csc(2, 2, [0, 2], [0, 0])


@pytest.mark.parametrize("size,T", [((300, 470, 60, 250), 24), ((1354, 1991, 260, 1137), 6)])
def test_synthetic_vs_oracle(gpu, size, T):
    raw = synthetic_case(*size, seed=17, parallel_lines=5, shared_gens=7)
    net = raw.network()
    from paper_2405_14032_b200.opf import load_profile
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    orc = B.OracleModel(net, T, scale)
    assert [nlp.sizes.n_vars, nlp.sizes.n_cons, nlp.sizes.jac_nnz, nlp.sizes.hess_nnz] == \
        orc.sizes[:4]
    for a, b in zip((*nlp.jac_structure(), *nlp.hess_structure()), orc.structure()):
        assert_bitexact(a, b)
    xl, xu, xs, _, _ = orc.bounds()
    x = interior_point(xl, xu, xs, 3)
    w = row_weights(orc.sizes[1], 4, zero_every=13)
    for name, args in [("eval_f", (x,)), ("eval_grad", (x,)), ("eval_g", (x,)),
                       ("eval_jac", (x,)), ("eval_hess", (x, w, 1.0))]:
        okg, got = getattr(nlp, name)(*args)
        oko, ref, _ = getattr(orc, name)(*args)
        assert okg and oko
        assert_close(np.atleast_1d(got), np.atleast_1d(ref), what=name)
    nlp.lift(1e-4)
    lo = orc.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    OK = orc.kkt()
    for a, b in zip(K.structure(), OK.structure()):
        assert_bitexact(a, b)
    _, jv, _ = orc.eval_jac(x)
    _, hv, _ = orc.eval_hess(x, w, 1.0)
    sx, ss = sigmas(len(lo["free_to_full"]), orc.sizes[1], 5)
    K.set_jacobian(jv, mem=GN_IN_FULL)
    OK.set_jacobian(jv[lo["jac_pick"]])
    for dw, dc in DELTAS:
        K.assemble(hv, sx, ss, dw, dc, mem=GN_IN_FULL)
        OK.assemble(hv[lo["hess_pick"]], sx, ss, dw, dc)
        for a, b in zip(K.values(), OK.values()):
            assert_bitexact(a, b)


def _edge_network(seed=21):
    """Parallel lines, several generators per bus, fixed generators (pmin == pmax,
    qmin == qmax) and fixed voltages (vmin == vmax): every lifted-filter branch."""
    raw = synthetic_case(400, 640, 90, 330, seed=seed, parallel_lines=9, shared_gens=12)
    net = raw.network()
    net.gen_pmin[3] = net.gen_pmax[3]
    net.gen_qmin[7] = net.gen_qmax[7]
    net.gen_pmin[11] = net.gen_pmax[11]
    net.gen_qmin[11] = net.gen_qmax[11]
    for b in (5, 17, 200):
        net.bus_vmin[b] = net.bus_vmax[b]
    net.gen_ramp[20] = np.inf  # a non-ramping generator
    net.line_smax[[2, 50, 51]] = np.inf  # unrated lines
    return net


@pytest.mark.parametrize("T", [1, 2, 7])
def test_specialised_kkt_equals_generic_and_oracle(gpu, T):
    from paper_2405_14032_b200.opf import load_profile
    net = _edge_network()
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    assert K.opf_ready == 1, "specialised enumeration did not verify"
    orc = B.OracleModel(net, T, scale)
    lo = orc.lift(1e-4)
    assert nlp.sizes.n_free == len(lo["free_to_full"])
    xl, xu, xs, _, _ = orc.bounds()
    x = interior_point(xl, xu, xs, 9)
    w = row_weights(orc.sizes[1], 10, zero_every=7)
    _, jv, _ = orc.eval_jac(x)
    _, hv, _ = orc.eval_hess(x, w, 1.0)
    sx, ss = sigmas(len(lo["free_to_full"]), orc.sizes[1], 12)
    OK = orc.kkt()
    OK.set_jacobian(jv[lo["jac_pick"]])
    for algo in (2, 1):  # specialised, then generic contributor lists
        K.set_algorithm(algo)
        K.set_jacobian(jv, mem=GN_IN_FULL)
        for dw, dc in DELTAS:
            K.assemble(hv, sx, ss, dw, dc, mem=GN_IN_FULL)
            OK.assemble(hv[lo["hess_pick"]], sx, ss, dw, dc)
            for a, b, nm in zip(K.values(), OK.values(), ("A", "M")):
                assert_bitexact(a, b, f"{nm} algo={algo} dw={dw}")


def _fused_check(nlp, K, x, w, ow, sx, ss):
    """Fused A/M (from x) == set_jacobian(eval_jac(x)) / assemble(eval_hess(x, w, ow))."""
    assert K.fused_ready == 1, "fused enumeration did not verify"
    ok, jv = nlp.eval_jac(x)
    ok2, hv = nlp.eval_hess(x, w, ow)
    assert ok and ok2
    K.set_jacobian(jv, mem=GN_IN_FULL)
    for dw, dc in DELTAS:
        K.assemble(hv, sx, ss, dw, dc, mem=GN_IN_FULL)
        a_ref, m_ref = K.values()
        K.set_jacobian_x(x)
        K.assemble_x(x, w, ow, sx, ss, dw, dc)
        a, m = K.values()
        assert_bitexact(a, a_ref, f"fused A dw={dw}")
        assert_bitexact(m, m_ref, f"fused M dw={dw}")
        # gn_kkt_update_x (set_jacobian_x + assemble_x in one pass) over poisoned A / M
        K.set_jacobian(np.full_like(jv, np.nan), mem=GN_IN_FULL)
        K.assemble(np.full_like(hv, np.nan), sx, ss, dw, dc, mem=GN_IN_FULL)
        K.update_x(x, w, ow, sx, ss, dw, dc)
        a, m = K.values()
        assert_bitexact(a, a_ref, f"update_x A dw={dw}")
        assert_bitexact(m, m_ref, f"update_x M dw={dw}")
        K.set_jacobian(jv, mem=GN_IN_FULL)  # restore the contract A for the next delta


@pytest.mark.parametrize("fx", FIXTURES)
def test_fused_kkt_equals_contract_path_fixtures(gpu, fx):
    nlp, z, meta, net = _nlp(fx)
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    _fused_check(nlp, K, z["x"], z["w"], float(z["ow"]), z["sx"], z["ss"])
    # and against the reference's own M (value tolerance: H/J differ by sin/cos ulps)
    K.set_jacobian_x(z["x"])
    K.assemble_x(z["x"], z["w"], float(z["ow"]), z["sx"], z["ss"], *DELTAS[1])
    assert_close(K.values()[1], z["mvals1"], what="fused M vs reference")


@pytest.mark.parametrize("T", [1, 2, 7, 40])
def test_fused_kkt_equals_contract_path_edge_network(gpu, T):
    from paper_2405_14032_b200.opf import load_profile
    net = _edge_network(seed=30 + T)
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, T)
    w = row_weights(nlp.sizes.n_cons, T + 1, zero_every=9)
    sx, ss = sigmas(nlp.sizes.n_free, nlp.sizes.n_cons, T + 2)
    _fused_check(nlp, K, x, w, 0.7, sx, ss)
    _fused_check(nlp, K, x, w, 0.0, sx, ss)  # restoration-style obj_weight 0


def test_stream_switching_any_order(gpu):
    """set_stream on the context, then on a KKT created before it (which still
    referenced the context's own stream), then back to the own streams."""
    import torch
    from paper_2405_14032_b200.opf import load_profile
    raw = synthetic_case(60, 100, 15, 50, seed=9)
    net = raw.network()
    nlp = OpfNlp(net, 3, load_profile(net.n_load, 3))
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    st = torch.cuda.Stream()
    nlp.set_stream(st.cuda_stream)
    K.set_stream(st.cuda_stream)
    xl, xu, xs, _, _ = nlp.bounds()
    ok, g1 = nlp.eval_g(xs)
    assert ok
    nlp.reset_stream()
    K.reset_stream()
    ok, g2 = nlp.eval_g(xs)
    assert ok and np.array_equal(g1, g2)
    K.close()


def test_reset_stream_then_async_assemble(gpu):
    """a lifted KKT reset with set_stream(NULL) returns to its context's own
    stream (not the legacy default stream), so GN_MEM_DEVICE_ASYNC work stays ordered
    after the callbacks; torch's default stream (handle 0) is the legacy stream, not a
    reset."""
    import torch
    from paper_2405_14032_b200.abi import GN_IN_FULL, GN_MEM_DEVICE_ASYNC
    from paper_2405_14032_b200.opf import load_profile
    raw = synthetic_case(60, 100, 15, 50, seed=19)
    net = raw.network()
    nlp = OpfNlp(net, 4, load_profile(net.n_load, 4))
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    K.reset_stream()
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 3)
    w = row_weights(nlp.n_cons(), 4)
    sx, ss = sigmas(nlp.sizes.n_free, nlp.n_cons(), 5)
    ok, jv = nlp.eval_jac(x)
    ok2, hv = nlp.eval_hess(x, w, 1.0)
    assert ok and ok2
    K.set_jacobian(jv, mem=GN_IN_FULL)
    K.assemble(hv, sx, ss, 0.0, 0.0, mem=GN_IN_FULL)
    a_ref, m_ref = K.values()
    dev = torch.device("cuda", 0)
    dx = torch.from_numpy(x).to(dev)
    dJ = torch.empty(nlp.sizes.jac_nnz, dtype=torch.float64, device=dev)
    dH = torch.empty(nlp.sizes.hess_nnz, dtype=torch.float64, device=dev)
    dw_, dsx, dss = (torch.from_numpy(a).to(dev) for a in (w, sx, ss))
    torch.cuda.synchronize()
    for _ in range(3):  # callbacks then the KKT, all async on the context's stream
        nlp.eval_device("jac", dx, dJ, sync=False)
        nlp.eval_device("hess", dx, dH, w=dw_, ow=1.0, sync=False)
        K.set_jacobian(dJ, mem=GN_MEM_DEVICE_ASYNC | GN_IN_FULL)
        K.assemble(dH, dsx, dss, 0.0, 0.0, mem=GN_MEM_DEVICE_ASYNC | GN_IN_FULL)
        a, m = K.values()
        assert np.array_equal(a, a_ref) and np.array_equal(m, m_ref)
        dJ.zero_()
        dH.zero_()
        torch.cuda.synchronize()  # the zero fills run on torch's stream
    # torch's default stream (handle 0) is the legacy stream, not a reset
    nlp.set_stream(torch.cuda.default_stream(dev).cuda_stream)
    ok, g1 = nlp.eval_g(x)
    nlp.reset_stream()
    ok2, g2 = nlp.eval_g(x)
    assert ok and ok2 and np.array_equal(g1, g2)
    K.close()


def test_line_search_trial_fg(gpu):
    """gn_eval_fg: f and g of a trial point in one call, bit-identical
    to eval_f + eval_g; a failure reports the first failing (pattern, record) of
    the pair, as the reference's eval_f-then-eval_g does."""
    nlp, z, meta, net = _nlp("synth_T3")
    ok, f, g = nlp.eval_fg(z["x"])
    okf, fr = nlp.eval_f(z["x"])
    okg, gr = nlp.eval_g(z["x"])
    assert ok and okf and okg
    assert f == fr and np.array_equal(g, gr)
    orc = B.OracleModel(net, meta["periods"], z["scale"])
    n = meta["sizes"][0]
    for idx in (n // 2, 5):  # a flow (g fails), a generator (f fails first)
        xb = z["x"].copy()
        xb[idx] = np.nan
        ok, _, _ = nlp.eval_fg(xb)
        oko, _, failf = orc.eval_f(xb)
        okg, _, failg = orc.eval_g(xb)
        assert ok == (oko and okg)
        assert nlp.last_error == (failf if not oko else failg)


def test_fused_kkt_isolated_and_high_degree_buses(gpu):
    """Buses outside the register-resident classes: an isolated bus (no lines; its
    v/th columns hold only dw + Sx) and a hub of degree 9 (slot-program class), next
    to parallel lines; fused == contract bit for bit, and the contract path == oracle."""
    from paper_2405_14032_b200.network import RawCase
    from paper_2405_14032_b200.opf import load_profile
    raw = synthetic_case(80, 130, 20, 60, seed=23, parallel_lines=3, shared_gens=2)
    bus, gen, br, gc = raw.bus.copy(), raw.gen.copy(), raw.branch.copy(), raw.gencost.copy()
    nb = int(bus[:, 0].max())
    iso = bus[5].copy()
    iso[0], iso[1] = nb + 1, 1  # a PQ bus with the load of bus 6 and no branch
    bus = np.vstack([bus, iso])
    g = gen[0].copy()
    g[0] = nb + 1
    gen = np.vstack([gen, g])
    gc = np.vstack([gc, gc[0]])
    hub = int(bus[10, 0])
    extra = []
    for k in range(7):  # degree 2 + 7 chords = 9 at the hub
        row = br[0].copy()
        row[0], row[1] = hub, int(bus[(20 + 7 * k) % 80, 0])
        extra.append(row)
    br = np.vstack([br] + extra)
    raw2 = RawCase(raw.base_mva, bus, gen, br, gc)
    net = raw2.network()
    T = 5
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 31)
    w = row_weights(nlp.sizes.n_cons, 32, zero_every=6)
    sx, ss = sigmas(nlp.sizes.n_free, nlp.sizes.n_cons, 33)
    _fused_check(nlp, K, x, w, 0.9, sx, ss)
    orc = B.OracleModel(net, T, scale)
    lo = orc.lift(1e-4)
    Ko = orc.kkt()
    ok, jv, _ = orc.eval_jac(x)
    ok2, hv, _ = orc.eval_hess(x, w, 0.9)
    Ko.set_jacobian(jv[lo["jac_pick"]])
    Ko.assemble(hv[lo["hess_pick"]], sx, ss, *DELTAS[1])
    K.update_x(x, w, 0.9, sx, ss, *DELTAS[1])
    a, m = K.values()
    a_o, m_o = Ko.values()
    assert_close(m, m_o, what="fused M vs oracle (sin/cos ulps)")
    assert_close(a, a_o, what="fused A vs oracle")


def test_degree_above_32_falls_back_loudly(gpu):
    """A bus with more than 32 lines exceeds the fused kernels' one-line-per-lane
    layout: the fused path reports GN_ERR_UNSUPPORTED (never a silent wrong answer)
    and the contract KKT still matches the oracle."""
    from paper_2405_14032_b200.network import RawCase
    from paper_2405_14032_b200.opf import load_profile
    raw = synthetic_case(120, 200, 25, 90, seed=29)
    br = raw.branch.copy()
    hub = int(raw.bus[3, 0])
    extra = []
    for k in range(34):
        row = br[0].copy()
        row[0], row[1] = hub, int(raw.bus[(10 + 3 * k) % 120, 0])
        if row[1] != hub:
            extra.append(row)
    raw2 = RawCase(raw.base_mva, raw.bus, raw.gen, np.vstack([br] + extra), raw.gencost)
    net = raw2.network()
    T = 3
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    assert K.fused_ready == 0
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 41)
    w = row_weights(nlp.sizes.n_cons, 42)
    sx, ss = sigmas(nlp.sizes.n_free, nlp.sizes.n_cons, 43)
    with pytest.raises(GridError) as e:
        K.update_x(x, w, 1.0, sx, ss, *DELTAS[1])
    assert e.value.code == 4  # GN_ERR_UNSUPPORTED
    ok, jv = nlp.eval_jac(x)
    ok2, hv = nlp.eval_hess(x, w, 1.0)
    K.set_jacobian(jv, mem=GN_IN_FULL)
    K.assemble(hv, sx, ss, *DELTAS[1], mem=GN_IN_FULL)
    a, m = K.values()
    orc = B.OracleModel(net, T, scale)
    lo = orc.lift(1e-4)
    Ko = orc.kkt()
    ok, jo, _ = orc.eval_jac(x)
    ok2, ho, _ = orc.eval_hess(x, w, 1.0)
    Ko.set_jacobian(jo[lo["jac_pick"]])
    Ko.assemble(ho[lo["hess_pick"]], sx, ss, *DELTAS[1])
    a_o, m_o = Ko.values()
    assert_close(m, m_o, what="M (fallback) vs oracle")
    assert_close(a, a_o, what="A (fallback) vs oracle")


@pytest.mark.parametrize("T", [1, 3])
def test_no_thermal_no_ramp_patterns(gpu, T):
    """Empty pattern blocks: every line unrated (no thermal rows, LT = 0) and no ramping
    generator (GR = 0) -- the pattern ids shift; callbacks, failure ids
    and the fused KKT must follow."""
    from paper_2405_14032_b200.opf import load_profile
    raw = synthetic_case(70, 110, 15, 50, seed=37, parallel_lines=2)
    net = raw.network()
    net.line_smax[:] = np.inf
    net.gen_ramp[:] = np.inf
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    orc = B.OracleModel(net, T, scale)
    assert [nlp.sizes.n_vars, nlp.sizes.n_cons, nlp.sizes.jac_nnz, nlp.sizes.hess_nnz] == \
        orc.sizes[:4]
    assert nlp.sizes.n_thermal == 0 and nlp.sizes.n_ramp_gens == 0
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 51)
    w = row_weights(nlp.sizes.n_cons, 52, zero_every=4)
    for name, args in [("eval_g", (x,)), ("eval_jac", (x,)), ("eval_hess", (x, w, 0.6))]:
        ok, v = getattr(nlp, name)(*args)
        oko, vo, _ = getattr(orc, name)(*args)
        assert ok and oko
        assert_close(v, vo, what=name)
    xb = x.copy()
    xb[len(x) // 2] = np.nan  # a flow variable: the failing pattern id shifts with LT = 0
    ok, _ = nlp.eval_g(xb)
    oko, _, fail = orc.eval_g(xb)
    assert not ok and not oko and nlp.last_error == fail
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    sx, ss = sigmas(nlp.sizes.n_free, nlp.sizes.n_cons, 53)
    _fused_check(nlp, K, x, w, 0.6, sx, ss)


@pytest.mark.parametrize("order", [(0, 1, 2), (2, 1, 0), (1, 0, 2), (0, 2, 1)])
def test_destroy_order_any(gpu, order):
    """Context, KKT and IPM objects may be destroyed in any order (a garbage collector
    finalising a reference cycle does): a destroyed object that others were built on
    stays alive until the last of them goes, and the survivors keep working."""
    import torch
    from paper_2405_14032_b200.opf import Ipm, load_profile
    raw = synthetic_case(40, 60, 8, 30, seed=3)
    net = raw.network()
    nlp = OpfNlp(net, 3, load_profile(net.n_load, 3))
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    st = nlp.lifted_structure()
    xl, xu, xs, _, _ = nlp.bounds()
    f2f = st["free_to_full"]
    ipm = Ipm(K, xl[f2f], xu[f2f], st["s_lower"], st["s_upper"])
    objs = [nlp, K, ipm]
    x = interior_point(xl, xu, xs, 5)
    for i in order:
        objs[i].close()
        if not isinstance(objs[1], CondensedKkt) or objs[1].h is None:
            continue
        if objs[1].fused_ready and objs[1].h is not None:  # the KKT still works
            w = row_weights(nlp.sizes.n_cons, 6)
            sx, ss = sigmas(nlp.sizes.n_free, nlp.sizes.n_cons, 7)
            objs[1].update_x(x, w, 1.0, sx, ss, *DELTAS[0])
    torch.cuda.synchronize()


@pytest.mark.parametrize("seed", range(int(os.environ.get("GN_TEST_SEEDS", "8"))))
def test_fused_kkt_randomised_networks(gpu, seed):
    """Randomised sweep: network size, parallel lines, shared generators, fixed
    generators / voltages, unrated lines and horizon length (partial 32-period chunks)
    -- the fused A/M must equal the contract path bit for bit every time."""
    from paper_2405_14032_b200.opf import load_profile
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.integers(20, 200))
    L = N + int(rng.integers(N // 3, N))
    G = int(rng.integers(3, max(4, N // 4)))
    D = int(rng.integers(N // 3, N))
    raw = synthetic_case(N, L, G, D, seed=int(rng.integers(1, 10_000)),
                         parallel_lines=int(rng.integers(0, 4)),
                         shared_gens=int(rng.integers(0, 4)))
    net = raw.network()
    for g in rng.choice(net.n_gen, size=min(2, net.n_gen), replace=False):
        net.gen_pmin[g] = net.gen_pmax[g]
    for b in rng.choice(net.n_bus, size=2, replace=False):
        if b != net.reference_bus:
            net.bus_vmin[b] = net.bus_vmax[b]
    net.line_smax[rng.random(net.n_line) < 0.2] = np.inf
    net.gen_ramp[rng.random(net.n_gen) < 0.2] = np.inf
    T = int(rng.integers(1, 70))
    scale = load_profile(net.n_load, T)
    nlp = OpfNlp(net, T, scale)
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, seed)
    w = row_weights(nlp.sizes.n_cons, seed + 1, zero_every=int(rng.integers(2, 9)))
    sx, ss = sigmas(nlp.sizes.n_free, nlp.sizes.n_cons, seed + 2)
    ow = float(rng.uniform(0, 2))
    _fused_check(nlp, K, x, w, ow, sx, ss)
    # and the callbacks / structures against the bit-exact C restatement
    orc = B.OracleModel(net, T, scale)
    for a, b in zip(orc.structure(), (*nlp.jac_structure(), *nlp.hess_structure())):
        assert_bitexact(a, b, "structure")
    for name, args in [("eval_g", (x,)), ("eval_jac", (x,)), ("eval_hess", (x, w, ow))]:
        ok, v = getattr(nlp, name)(*args)
        oko, vo, _ = getattr(orc, name)(*args)
        assert ok and oko
        assert_close(v, vo, what=name)


@pytest.mark.parametrize("T", [40, 96])
def test_bitwise_reproducible_across_launch_shapes(gpu, T):
    """Outputs are bitwise independent of the launch configuration and of repetition
    (pattern_model.hpp:270-273): KKT grid caps (grid-stride virtual CTAs), the bus-class
    lanes chosen for the size, and repeated calls (the objective's last-block sum)."""
    from paper_2405_14032_b200.opf import load_profile
    raw = synthetic_case(400, 620, 90, 330, seed=17, parallel_lines=3, shared_gens=3)
    net = raw.network()
    nlp = OpfNlp(net, T, load_profile(net.n_load, T))
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, T + 5)
    w = row_weights(nlp.sizes.n_cons, T + 6, zero_every=7)
    sx, ss = sigmas(nlp.sizes.n_free, nlp.sizes.n_cons, T + 7)
    ref = None
    for cap in (0, 1, 2, 3, 0):
        K.set_grid_cap(cap)
        K.update_x(x, w, 1.0, sx, ss, *DELTAS[1])
        a, m = K.values()
        if ref is None:
            ref = (a.copy(), m.copy())
        assert_bitexact(a, ref[0], f"A cap={cap}")
        assert_bitexact(m, ref[1], f"M cap={cap}")
    outs = []
    for _ in range(3):
        ok, f = nlp.eval_f(x)
        ok2, fg_f, fg_g = nlp.eval_fg(x)
        ok3, h = nlp.eval_hess(x, w, 1.0)
        assert ok and ok2 and ok3 and f == fg_f
        outs.append((f, fg_g, h))
    for f, g, h in outs[1:]:
        assert f == outs[0][0]
        assert np.array_equal(g, outs[0][1]) and np.array_equal(h, outs[0][2])
    K.close()


@pytest.mark.parametrize("fx", FIXTURES)
def test_eval_fg_matches_golden(gpu, fx):
    """gn_eval_fg values against the reference's own f and g at the golden point
    (fg was only compared with this repository's eval_f/eval_g)."""
    nlp, z, meta, net = _nlp(fx)
    ok, f, g = nlp.eval_fg(z["x"])
    assert ok
    assert_close([f], [float(z["f"])], what="fg: f")
    assert_close(g, z["g"], what="fg: g")
    bal = _bal_rows(meta, net)
    assert_bitexact(g[bal], z["g"][bal], "fg: balance rows (canonical order)")


@pytest.mark.parametrize("fx", FIXTURES)
@pytest.mark.parametrize("mem", ["host", "device"])
def test_lifted_gather_matches_reference(gpu, fx, mem):
    """gn_lifted_gather_{jac,hess} (LiftedProblem::eval_jac/eval_hess picks, lifted.hpp:
    128-159): the reference's full J / H values gathered equal the reference's own lifted
    values bit for bit, through host and device pointers."""
    import torch
    nlp, z, meta, net = _nlp(fx)
    nlp.lift(1e-4)
    for which, full, lifted in (("jac", z["jac"], z["jac_l"]), ("hess", z["hess"], z["hess_l"])):
        if mem == "host":
            got = nlp.lifted_gather(which, full)
        else:
            dev = torch.device("cuda", 0)
            out = torch.full((len(lifted),), np.nan, dtype=torch.float64, device=dev)
            nlp.lifted_gather(which, torch.from_numpy(full).to(dev), out=out, mem=GN_MEM_DEVICE)
            got = out.cpu().numpy()
        assert_bitexact(got, lifted, f"lifted {which} gather")


def test_values_ptr_views_the_kkt_arrays(gpu):
    """gn_kkt_values_ptr: zero-copy views of the KKT's own A and M equal gn_kkt_values."""
    import torch

    class _View:
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                             "data": (ptr, False), "version": 3}

    nlp, z, meta, net = _nlp("case118_T4")
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    dw, dc = DELTAS[1]
    K.update_x(z["x"], z["w"], float(z["ow"]), z["sx"], z["ss"], dw, dc)
    a, m = K.values()
    pa, pm = K.values_ptr()
    assert pa and pm
    dev = torch.device("cuda", 0)
    torch.cuda.synchronize()
    assert_bitexact(torch.as_tensor(_View(pa, K.a_nnz), device=dev).cpu().numpy(), a, "A view")
    assert_bitexact(torch.as_tensor(_View(pm, K.m_nnz), device=dev).cpu().numpy(), m, "M view")


@pytest.mark.parametrize("fx", ["case9_T2", "case118_T4", "synth_T3"])
def test_eval_all_equals_the_five_callbacks(gpu, fx):
    """gn_eval_all (one launch) writes exactly what eval_f / grad / g / jac / hess write, and
    reports the same first failure."""
    nlp, z, meta, net = _nlp(fx)
    x, w, ow = z["x"], z["w"], float(z["ow"])
    ok, (f, grad, g, jac, hess) = nlp.eval_all(x, w, ow)
    assert ok
    assert f[0] == nlp.eval_f(x)[1]
    assert_bitexact(grad, nlp.eval_grad(x)[1], "grad")
    assert_bitexact(g, nlp.eval_g(x)[1], "g")
    assert_bitexact(jac, nlp.eval_jac(x)[1], "jac")
    assert_bitexact(hess, nlp.eval_hess(x, w, ow)[1], "hess")
    assert_close(hess, z["hess"], what="hess vs reference")
    xb = x.copy()
    xb[len(x) // 2] = np.nan
    firsts = []
    for name, args in [("eval_f", (xb,)), ("eval_grad", (xb,)), ("eval_g", (xb,)),
                       ("eval_jac", (xb,)), ("eval_hess", (xb, w, ow))]:
        okc, _ = getattr(nlp, name)(*args)
        if not okc:
            firsts.append(nlp.last_error)
    ok, _ = nlp.eval_all(xb, w, ow)
    assert ok == (not firsts)
    if firsts:
        assert nlp.last_error == min(firsts)


def test_values_start_overlaps_and_orders_before_the_next_write(gpu):
    """gn_kkt_values_start: the side-stream read-back of A / M into pinned memory lands the
    values of the moment it was started -- the next assemble / set_jacobian waits for it on
    the device -- and equals the synchronous read-back."""
    import torch
    nlp, z, meta, net = _nlp("case118_T4")
    nlp.lift(1e-4)
    K = CondensedKkt(nlp=nlp)
    (dw, dc), (dw2, dc2) = DELTAS[0], DELTAS[1]
    K.update_x(z["x"], z["w"], float(z["ow"]), z["sx"], z["ss"], dw, dc)
    a_ref, m_ref = K.values()
    pa = torch.full((K.a_nnz,), np.nan, dtype=torch.float64).pin_memory()
    pm = torch.full((K.m_nnz,), np.nan, dtype=torch.float64).pin_memory()
    K.values_start(pa, pm)
    # a different assembly right behind it (host inputs): its kernels must not overtake the copy
    K.update_x(z["x"] * 1.01, z["w"], float(z["ow"]), z["sx"], z["ss"], dw2, dc2)
    K.values_wait()
    assert_bitexact(pa.numpy(), a_ref, "A read back before the next write")
    assert_bitexact(pm.numpy(), m_ref, "M read back before the next write")
    a2, m2 = K.values()
    assert not np.array_equal(m2, m_ref)  # the second assembly did change M
    K.values_start(pa, None)
    K.values_wait()
    assert_bitexact(pa.numpy(), a2, "A after the second assembly")
