"""CPU: pin the oracle (oracle/gn_oracle.c) against the reference.

* bit-exact against the golden fixtures the UNMODIFIED reference produced
  (tests/golden/make_golden.py), for structures, bounds, every callback,
  the lifted filter and the condensed KKT;
* the reference's own known-answer tests (test_sparse.cpp:95-111,
  test_power.cpp:238-284, README.md:118-121, SURVEY Appendix B probe 1);
* when oracle/_ref is present (build container), bit-exact against the live
  reference on random synthetic networks, including failure reports.
"""
import numpy as np
import pytest

from helpers import (DELTAS, assert_bitexact, golden_eval, golden_meta, golden_network,
                     interior_point, row_weights, sigmas)
from oracle import bindings as B

FIXTURES = list(golden_meta()["fixtures"])


def _model(fx):
    meta = golden_meta()["fixtures"][fx]
    z = golden_eval(fx)
    net = golden_network(meta["case"])
    return B.OracleModel(net, meta["periods"], z["scale"]), z, meta


@pytest.mark.parametrize("fx", FIXTURES)
def test_oracle_matches_reference_fixture(fx):
    m, z, meta = _model(fx)
    assert m.sizes == meta["sizes"]
    for got, key in zip(m.bounds(), ("xl", "xu", "xs", "rl", "ru")):
        assert_bitexact(got, z[key], key)
    for got, key in zip(m.structure(), ("jr", "jc", "hr", "hc")):
        assert_bitexact(got, z[key], key)
    x, w, ow = z["x"], z["w"], float(z["ow"])
    ok, f, _ = m.eval_f(x)
    assert ok and f == float(z["f"])
    for name, args, key in [("eval_grad", (x,), "grad"), ("eval_g", (x,), "g"),
                            ("eval_jac", (x,), "jac"), ("eval_hess", (x, w, ow), "hess")]:
        ok, got, _ = getattr(m, name)(*args)
        assert ok
        assert_bitexact(got, z[key], key)


@pytest.mark.parametrize("fx", FIXTURES)
def test_oracle_lifted_and_kkt_match_reference_fixture(fx):
    m, z, meta = _model(fx)
    lift = m.lift(1e-4)
    assert list(m.lifted_sizes) == meta["lifted"]
    for k in ("free_to_full", "jac_rows", "jac_cols", "hess_rows", "hess_cols", "s_lower",
              "s_upper"):
        assert_bitexact(lift[k], z["l_" + k], k)
    # pick maps reproduce LiftedProblem's gathered values (lifted.hpp:249-264)
    assert_bitexact(z["jac"][lift["jac_pick"]], z["jac_l"], "jac pick")
    assert_bitexact(z["hess"][lift["hess_pick"]], z["hess_l"], "hess pick")
    K = m.kkt()
    assert [K.dim, K.a_nnz, K.m_nnz] == meta["kkt"]
    for got, key in zip(K.structure(), ("rowptr", "colidx", "colptr", "rowidx")):
        assert_bitexact(got, z[key], key)
    K.set_jacobian(z["jac_l"])
    for i, (dw, dc) in enumerate(DELTAS):
        K.assemble(z["hess_l"], z["sx"], z["ss"], dw, dc)
        a, mv = K.values()
        assert_bitexact(a, z["avals"], "A values")
        assert_bitexact(mv, z[f"mvals{i}"], f"M values delta#{i}")


def test_compress_to_csc_known_answer():
    # test_sparse.cpp:95-111
    cp, ri, sm = B.oracle_compress_to_csc(3, 2, [0, 1, 0, 2], [0, 0, 0, 1])
    assert cp.tolist() == [0, 2, 3] and ri.tolist() == [0, 1, 2] and sm.tolist() == [0, 1, 0, 2]
    K = B.OracleKkt(1, 0, [], [], [], [])  # degenerate: 1 variable, no rows
    assert K.m_nnz == 1
    with pytest.raises(ValueError):
        B.oracle_compress_to_csc(2, 2, [0, 2], [0, 0])


def test_model_dimension_known_answers():
    net = golden_network("case9")
    for T in (1, 2, 10, 30):  # test_power.cpp:238-284
        m = B.OracleModel(net, T, np.ones((T, net.n_load)))
        assert m.sizes[0] == 42 * T
        assert m.sizes[1] == 54 * T + 3 * (T - 1)
        assert m.sizes[4] == 9  # all nine lines rated
        assert m.sizes[5] == (3 if T >= 2 else 0)
    meta = golden_meta()
    net = golden_network("case118")
    m = B.OracleModel(net, 168, np.ones((168, net.n_load)))
    assert m.sizes[:4] == meta["case118_T168"]["sizes"][:4] == [120288, 173658, 598644, 1304190]
    m.lift(1e-4)
    assert list(m.lifted_sizes) == meta["case118_T168"]["lifted"]
    assert m.lifted_sizes[2:] == (595620, 1292094)


def test_pattern_offsets_closed_form():
    """SURVEY Appendix A.2 closed-form offsets (verified against freeze)."""
    net = golden_network("case30")
    T = 3
    m = B.OracleModel(net, T, np.ones((T, net.n_load)))
    jo, ho, rec = m.offsets()
    L, G, LT = net.n_line, net.n_gen, 41
    assert jo[1:12] == [0, 2 * L * T, 4 * L * T, 4 * L * T + G * T, 4 * L * T + 2 * G * T,
                        4 * L * T + 2 * G * T, 4 * L * T + 2 * G * T, 9 * L * T + 2 * G * T,
                        14 * L * T + 2 * G * T, 14 * L * T + 2 * G * T + 2 * LT * T,
                        16 * L * T + 2 * G * T + 2 * LT * T]
    assert ho[0:12] == [0, G * T, G * T + 2 * L * T, G * T + 4 * L * T, 2 * G * T + 4 * L * T,
                        3 * G * T + 4 * L * T, 3 * G * T + 4 * L * T, 3 * G * T + 4 * L * T,
                        3 * G * T + 19 * L * T, 3 * G * T + 34 * L * T,
                        3 * G * T + 34 * L * T + 3 * LT * T, 3 * G * T + 37 * L * T + 3 * LT * T]


# ------------------------------------------------------------- live reference
needs_ref = pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built here")


@needs_ref
@pytest.mark.parametrize("seed,T,par,shared", [(2, 2, 0, 0), (3, 3, 4, 3), (4, 5, 2, 6)])
def test_oracle_vs_live_reference_random(seed, T, par, shared):
    from paper_2405_14032_b200.network import synthetic_case
    raw = synthetic_case(25 + seed, 40 + 3 * seed, 7, 20, seed=seed, parallel_lines=par,
                         shared_gens=shared)
    text = raw.to_matpower()
    net = raw.network()
    assert net.equal(B.ref_parse_matpower(text)), "per-unit conversion differs from parser"
    scale = B.ref_load_profile(text, T, seed=seed)
    ref, orc = B.RefModel(text, T, scale), B.OracleModel(net, T, scale)
    assert ref.sizes == orc.sizes
    for a, b in zip(ref.structure(), orc.structure()):
        assert_bitexact(b, a)
    xl, xu, xs, _, _ = ref.bounds()
    x = interior_point(xl, xu, xs, seed)
    w = row_weights(ref.sizes[1], seed, zero_every=5)
    for name, args in [("eval_f", (x,)), ("eval_grad", (x,)), ("eval_g", (x,)),
                       ("eval_jac", (x,)), ("eval_hess", (x, w, 0.3))]:
        r, o = getattr(ref, name)(*args), getattr(orc, name)(*args)
        assert r[0] == o[0]
        assert_bitexact(np.atleast_1d(o[1]), np.atleast_1d(r[1]), name)
    # failure reports: a NaN in one flow variable and one voltage
    xb = x.copy()
    xb[ref.sizes[0] // 2] = np.nan
    xb[ref.sizes[0] - 3] = np.inf
    for name, args in [("eval_f", (xb,)), ("eval_grad", (xb,)), ("eval_g", (xb,)),
                       ("eval_jac", (xb,)), ("eval_hess", (xb, w, 0.3))]:
        r, o = getattr(ref, name)(*args), getattr(orc, name)(*args)
        assert r[0] == o[0], name
        assert r[2] == o[2], (name, r[2], o[2])
    lr, lo = ref.lift(1e-4), orc.lift(1e-4)
    for k in lr:
        assert_bitexact(lo[k], lr[k], k)
    ref.kkt_create()
    K = orc.kkt()
    for a, b in zip(ref.kkt_structure(), K.structure()):
        assert_bitexact(b, a)
    _, jv, _ = orc.eval_jac(x)
    _, hv, _ = orc.eval_hess(x, w, 1.0)
    sx, ss = sigmas(len(lo["free_to_full"]), ref.sizes[1], seed)
    jl, hl = jv[lo["jac_pick"]], hv[lo["hess_pick"]]
    ref.kkt_set_jacobian(jl)
    K.set_jacobian(jl)
    for dw, dc in DELTAS:
        ref.kkt_assemble(hl, sx, ss, dw, dc)
        K.assemble(hl, sx, ss, dw, dc)
        for a, b in zip(ref.kkt_values(), K.values()):
            assert_bitexact(b, a)
