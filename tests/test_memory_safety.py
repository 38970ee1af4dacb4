"""GPU: memory-safety evidence without compute-sanitizer (closed on this GPU pool: runs under
it left GPUs needing a reset).  Instead, every kernel family runs on buffers surrounded by
guard bands:

* inputs (x, w, sigma, J, H) sit between NaN guard bands: an out-of-bounds read turns an
  output into NaN, and the outputs are compared bit for bit with the unguarded call;
* outputs sit between guard bands holding a sentinel bit pattern, and are pre-filled with
  it: afterwards no guard word may have changed (no out-of-bounds write) and no output
  slot may still hold the sentinel (every contract slot rewritten on every call, SURVEY
  §8(d));
* the KKT's own A / M buffers carry a tail guard band (gn_debug_kkt_guard) checked the
  same way after the generic, OPF-contract, fused and published assemblies;
* shared-memory staging races would show as non-determinism: the fused assembly is run
  repeatedly, on several launch shapes, and must return identical bits.
"""
import numpy as np
import pytest
import torch

from helpers import DELTAS, golden_eval, golden_meta, golden_network, interior_point, row_weights, sigmas
from paper_2405_14032_b200.abi import GN_IN_FULL, GN_MEM_DEVICE
from paper_2405_14032_b200.opf import CondensedKkt, OpfNlp, load_profile

pytestmark = pytest.mark.gpu
G = 4096  # guard words on each side
SENT = 0x7FF4DEAD0000BEEF  # a NaN payload no kernel produces


def _dev():
    return torch.device("cuda", 0)


def guarded_in(a):
    """Device copy of `a` between NaN guard bands; returns (buffer, view)."""
    buf = torch.full((len(a) + 2 * G,), float("nan"), dtype=torch.float64, device=_dev())
    buf[G:G + len(a)] = torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(_dev())
    torch.cuda.synchronize()  # the library runs on its own (non-blocking) streams
    return buf, buf[G:G + len(a)]


def guarded_out(n):
    buf = torch.full((n + 2 * G,), SENT, dtype=torch.int64, device=_dev())
    torch.cuda.synchronize()
    return buf, buf[G:G + n].view(torch.float64)


def check_out(buf, n, what):
    bits = buf.cpu().numpy().view(np.uint64)
    assert np.all(bits[:G] == SENT) and np.all(bits[G + n:] == SENT), f"{what}: guard band written"
    assert not np.any(bits[G:G + n] == SENT), f"{what}: {int((bits[G:G + n] == SENT).sum())} slots never written"
    return bits[G:G + n].view(np.float64)


def _hub_network():
    from paper_2405_14032_b200.network import RawCase, synthetic_case
    raw = synthetic_case(80, 130, 20, 60, seed=23, parallel_lines=3, shared_gens=2)
    br = raw.branch.copy()
    hub = int(raw.bus[10, 0])
    extra = []
    for k in range(7):  # degree 9 at the hub: the slot-program bus class
        row = br[0].copy()
        row[0], row[1] = hub, int(raw.bus[(20 + 7 * k) % 80, 0])
        extra.append(row)
    return RawCase(raw.base_mva, raw.bus, raw.gen, np.vstack([br] + extra), raw.gencost).network()


def _problems():
    from test_gpu_parity import _edge_network
    meta = golden_meta()["fixtures"]["case9_T2"]
    yield "case9_T2", golden_network("case9"), 2, golden_eval("case9_T2")["scale"]
    net = _edge_network(seed=41)
    yield "edge_T5", net, 5, load_profile(net.n_load, 5)
    net = _hub_network()
    yield "hub_T37", net, 37, load_profile(net.n_load, 37)  # a partial 32-period chunk
    del meta


PROBLEMS = list(_problems())


@pytest.mark.parametrize("name,net,T,scale", PROBLEMS, ids=[p[0] for p in PROBLEMS])
def test_callbacks_guard_bands(gpu, name, net, T, scale):
    nlp = OpfNlp(net, T, scale)
    s = nlp.sizes
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 5)
    w = row_weights(s.n_cons, 6, zero_every=5)
    ref = {k: getattr(nlp, "eval_" + k)(x)[1] for k in ("grad", "g", "jac")}
    ref["hess"] = nlp.eval_hess(x, w, 0.9)[1]
    ref["f"] = np.array([nlp.eval_f(x)[1]])
    _, gx = guarded_in(x)
    _, gw = guarded_in(w)
    sizes = {"f": 1, "grad": s.n_vars, "g": s.n_cons, "jac": s.jac_nnz, "hess": s.hess_nnz}
    for k, n in sizes.items():
        buf, out = guarded_out(n)
        assert nlp.eval_device(k, gx, out, w=gw, ow=0.9)
        torch.cuda.synchronize()
        got = check_out(buf, n, k)
        assert np.array_equal(got, ref[k], equal_nan=False), f"{name} {k}"
    # the five in one call (gn_eval_all: one launch at these sizes)
    bufs = {k: guarded_out(n) for k, n in sizes.items()}
    ok, _ = nlp.eval_all(gx, gw, 0.9, outs=tuple(bufs[k][1] for k in ("f", "grad", "g", "jac",
                                                                        "hess")),
                         mem=GN_MEM_DEVICE)
    assert ok
    torch.cuda.synchronize()
    for k, n in sizes.items():
        assert np.array_equal(check_out(bufs[k][0], n, "all " + k), ref[k]), f"{name} all {k}"
    fb, fo = guarded_out(1)
    gb, go = guarded_out(s.n_cons)
    assert nlp.eval_device("fg", gx, (fo, go))
    torch.cuda.synchronize()
    assert check_out(fb, 1, "fg f")[0] == ref["f"][0]
    assert np.array_equal(check_out(gb, s.n_cons, "fg g"), ref["g"])
    nlp.lift(1e-4)
    s = nlp.sizes
    for which, full in (("jac", ref["jac"]), ("hess", ref["hess"])):
        n = s.jac_nnz_lifted if which == "jac" else s.hess_nnz_lifted
        _, gin = guarded_in(full)
        buf, out = guarded_out(n)
        nlp.lifted_gather(which, gin, out=out, mem=GN_MEM_DEVICE)
        torch.cuda.synchronize()
        assert np.array_equal(check_out(buf, n, "gather " + which), nlp.lifted_gather(which, full))
    # the lifted evaluations (gn_lifted_eval_*) on a guarded free-variable vector
    f2f = nlp.lifted_structure()["free_to_full"]
    _, gxf = guarded_in(x[f2f])
    for which, n in (("grad", s.n_free), ("g", s.n_cons), ("jac", s.jac_nnz_lifted),
                     ("hess", s.hess_nnz_lifted)):
        buf, out = guarded_out(n)
        ok, _ = nlp.lifted_eval(which, gxf, w=gw, ow=0.9, out=out, mem=GN_MEM_DEVICE)
        assert ok
        torch.cuda.synchronize()
        got = check_out(buf, n, "lifted " + which)
        want = nlp.lifted_eval(which, x[f2f], w=w, ow=0.9)[1]
        assert np.array_equal(got, want), f"{name} lifted {which}"


def _kkt_guard(K, fill):
    import ctypes as C
    out = (C.c_int64 * 4)()
    assert K.lib.gn_debug_kkt_guard(K.h, 1 if fill else 0, SENT, out) == 0
    return list(out)


@pytest.mark.parametrize("name,net,T,scale", PROBLEMS, ids=[p[0] for p in PROBLEMS])
def test_kkt_guard_bands_and_repeatability(gpu, name, net, T, scale):
    nlp = OpfNlp(net, T, scale)
    xl, xu, xs, _, _ = nlp.bounds()
    x = interior_point(xl, xu, xs, 7)
    w = row_weights(nlp.n_cons(), 8, zero_every=4)
    ok, J = nlp.eval_jac(x)
    ok2, H = nlp.eval_hess(x, w, 1.0)
    assert ok and ok2
    nlp.publish()  # lifts; a generic-array KKT on the same structure becomes "published"
    L = nlp.lifted_structure()
    sx, ss = sigmas(nlp.sizes.n_free, nlp.n_cons(), 9)
    _, gJ = guarded_in(J)
    _, gH = guarded_in(H)
    _, gJl = guarded_in(J[L["jac_pick"]])
    _, gHl = guarded_in(H[L["hess_pick"]])
    _, gsx = guarded_in(sx)
    _, gss = guarded_in(ss)
    _, gx = guarded_in(x)
    _, gw = guarded_in(w)
    Kl = CondensedKkt(nlp=nlp)
    assert Kl.fused_ready == 1
    Kg = CondensedKkt(nlp.sizes.n_free, nlp.n_cons(), L["jac_rows"], L["jac_cols"],
                      L["hess_rows"], L["hess_cols"])
    assert Kg.opf_ready == 1  # recognised through gn_ctx_publish
    Kg.set_algorithm(1)       # ... and forced onto the generic contributor-list kernels
    Kp = CondensedKkt(nlp.sizes.n_free, nlp.n_cons(), L["jac_rows"], L["jac_cols"],
                      L["hess_rows"], L["hess_cols"])
    for dw, dc in DELTAS:
        runs = {}
        for tag, K, fn in (
                ("generic", Kg, lambda K: (K.set_jacobian(gJl, mem=GN_MEM_DEVICE),
                                           K.assemble(gHl, gsx, gss, dw, dc, mem=GN_MEM_DEVICE))),
                ("published", Kp, lambda K: (K.set_jacobian(gJl, mem=GN_MEM_DEVICE),
                                             K.assemble(gHl, gsx, gss, dw, dc, mem=GN_MEM_DEVICE))),
                ("opf-full", Kl, lambda K: (K.set_jacobian(gJ, mem=GN_MEM_DEVICE | GN_IN_FULL),
                                            K.assemble(gH, gsx, gss, dw, dc,
                                                       mem=GN_MEM_DEVICE | GN_IN_FULL))),
                ("fused", Kl, lambda K: K.update_x(gx, gw, 1.0, gsx, gss, dw, dc,
                                                   mem=GN_MEM_DEVICE))):
            _kkt_guard(K, True)
            fn(K)
            torch.cuda.synchronize()
            assert _kkt_guard(K, False) == [0, 0, 0, 0], f"{name} {tag}: unwritten / guard words"
            runs[tag] = K.values()
        a0, m0 = runs["generic"]
        for tag, (a, m) in runs.items():
            assert np.array_equal(a, a0) and np.array_equal(m, m0), f"{name} {tag} vs generic"
        # repeatability of the fused (shared-memory staged) kernels across launch shapes
        for cap in (0, 1, 2, 3, 0, 2):
            Kl.set_grid_cap(cap)
            Kl.update_x(gx, gw, 1.0, gsx, gss, dw, dc, mem=GN_MEM_DEVICE)
            a, m = Kl.values()
            assert np.array_equal(a, a0) and np.array_equal(m, m0), f"{name} repeat cap={cap}"
    for K in (Kg, Kp, Kl):
        K.close()
