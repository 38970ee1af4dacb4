"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/make_golden.py               # everything (~6 min: reference solves)
    python tests/golden/make_golden.py --solves KEY  # networks + the named solves only
Writes tests/golden/networks.npz, eval_<name>.npz, meta.json.  The GPU box has
no /root/reference, so tests there read only these committed files.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import interior_point, row_weights, sigmas, DELTAS  # noqa: E402
from oracle import bindings as B  # noqa: E402
from paper_2405_14032_b200.network import CONFIG_SIZES, synthetic_case  # noqa: E402

OUT = Path(__file__).resolve().parent
DATA = Path("/root/reference/proj/data")

# (fixture name, network, T, resolution)
FIXTURES = [
    ("case9_T1", "case9", 1, 60.0),
    ("case9_T2", "case9", 2, 60.0),
    ("case30_T3", "case30", 3, 60.0),
    ("case118_T1", "case118", 1, 60.0),
    ("case118_T4", "case118", 4, 60.0),
    ("synth_T3", "synth", 3, 60.0),
]


def texts():
    t = {c: (DATA / f"{c}.m").read_text() for c in ("case9", "case30", "case118")}
    # edge-case network: parallel lines (both orientations) + several generators per bus
    t["synth"] = synthetic_case(40, 70, 12, 30, seed=5, parallel_lines=6,
                                shared_gens=5).to_matpower()
    # BASELINE configs[1] size (case1354pegase-size) for the end-to-end solve.  The config's
    # generator / load counts give less capacity than demand: at full demand the reference
    # IPM ends "infeasible" (84 iterations), at half demand it hits the iteration limit;
    # at 0.3 x demand it solves (36 iterations, ~47 s on this container's host)
    t["case1354s"] = synthetic_case(*CONFIG_SIZES["case1354pegase"], seed=1,
                                    load_scale=0.3).to_matpower()
    # self-loop lines (from bus == to bus; MATPOWER accepts them and the reference models
    # them as ordinary lines whose two voltage ends coincide)
    loop = synthetic_case(60, 95, 15, 45, seed=8, load_scale=0.5)
    loop.branch[5, 1] = loop.branch[5, 0]
    loop.branch[30, 0] = loop.branch[30, 1]
    t["synthloop"] = loop.to_matpower()
    # overloaded (1.3 x demand): the reference IPM enters feasibility restoration and ends
    # "infeasible" -- the restoration problem runs over the same seams
    t["synthinf"] = synthetic_case(40, 70, 12, 30, seed=1, load_scale=1.3).to_matpower()
    return t


# end-to-end reference solves (SURVEY §8(c) goldens), tol 1e-4: key -> (case, T, resolution)
SOLVES = {
    "case9_T1": ("case9", 1, 60.0),
    "case30_T30_r30": ("case30", 30, 30.0),
    "case118_T24": ("case118", 24, 60.0),
    "case118_T168": ("case118", 168, 60.0),        # 40 iterations
    "case1354s_T24": ("case1354s", 24, 60.0),      # SURVEY §7 step 7 (configs[1] size)
    "synthloop_T4": ("synthloop", 4, 60.0),        # two self-loop lines
    "synthinf_T3": ("synthinf", 3, 60.0),          # restoration, ends infeasible
}


def main():
    only = sys.argv[sys.argv.index("--solves") + 1:] if "--solves" in sys.argv else None
    T = texts()
    nets = {}
    for name, text in T.items():
        net = B.ref_parse_matpower(text)
        for k in net.F64 + net.I32:
            nets[f"{name}/{k}"] = getattr(net, k)
        nets[f"{name}/base_mva"] = np.array(net.base_mva)
        nets[f"{name}/reference_bus"] = np.array(net.reference_bus)
    np.savez_compressed(OUT / "networks.npz", **nets)
    if only is not None:
        meta = json.loads((OUT / "meta.json").read_text())
        for key in only:
            case, periods, res = SOLVES[key]
            scale = B.ref_load_profile(T[case], periods, resolution=res)
            r = B.RefModel(T[case], periods, scale).solve(1e-4)
            meta["solves"][key] = dict(case=case, periods=periods, resolution=res, **r)
            print(key, r)
        (OUT / "meta.json").write_text(json.dumps(meta, indent=1))
        return
    meta = {"fixtures": {}, "solves": {}}
    for fx, case, periods, res in FIXTURES:
        text = T[case]
        scale = B.ref_load_profile(text, periods, resolution=res)
        ref = B.RefModel(text, periods, scale)
        xl, xu, xs, rl, ru = ref.bounds()
        x = interior_point(xl, xu, xs)
        w = row_weights(ref.sizes[1], zero_every=11)
        ow = 1.0
        jr, jc, hr, hc = ref.structure()
        okf, f, _ = ref.eval_f(x)
        okg1, grad, _ = ref.eval_grad(x)
        okg, g, _ = ref.eval_g(x)
        okj, jac, _ = ref.eval_jac(x)
        okh, hess, _ = ref.eval_hess(x, w, ow)
        assert okf and okg1 and okg and okj and okh
        lift = ref.lift(1e-4)
        xfree = x[lift["free_to_full"]]
        jl = np.empty(len(lift["jac_rows"]))
        hl = np.empty(len(lift["hess_rows"]))
        assert ref.L.gnr_lifted_eval_jac(ref.h, B._f(xfree), B._f(jl))
        assert ref.L.gnr_lifted_eval_hess(ref.h, B._f(xfree), B._f(w), ow, B._f(hl))
        ksz = ref.kkt_create()
        rp, ci, cp, ri = ref.kkt_structure()
        sx, ss = sigmas(len(xfree), ref.sizes[1])
        out = dict(scale=scale, x=x, w=w, ow=np.array(ow), sx=sx, ss=ss, xl=xl, xu=xu, xs=xs,
                   rl=rl, ru=ru, jr=jr, jc=jc, hr=hr, hc=hc, f=np.array(f), grad=grad, g=g,
                   jac=jac, hess=hess, jac_l=jl, hess_l=hl, rowptr=rp, colidx=ci, colptr=cp,
                   rowidx=ri, **{f"l_{k}": v for k, v in lift.items()})
        ref.kkt_set_jacobian(jl)
        for i, (dw, dc) in enumerate(DELTAS):
            ref.kkt_assemble(hl, sx, ss, dw, dc)
            a, m = ref.kkt_values()
            out[f"avals"] = a
            out[f"mvals{i}"] = m
        np.savez_compressed(OUT / f"eval_{fx}.npz", **out)
        meta["fixtures"][fx] = dict(case=case, periods=periods, resolution=res,
                                    sizes=ref.sizes, lifted=list(ref.lifted_sizes),
                                    kkt=ksz[:3], factor_nnz=ksz[3])
        print(fx, ref.sizes, ref.lifted_sizes, ksz)
    # end-to-end reference solves (SURVEY §8(c) goldens), tol 1e-4
    for key, (case, periods, res) in SOLVES.items():
        text = T[case]
        scale = B.ref_load_profile(text, periods, resolution=res)
        r = B.RefModel(text, periods, scale).solve(1e-4)
        meta["solves"][key] = dict(case=case, periods=periods, resolution=res, **r)
        print(key, r)
    # size known-answers at case118 x 168 (README.md:118-121, SURVEY Appendix B probe 1)
    scale = B.ref_load_profile(T["case118"], 168)
    r = B.RefModel(T["case118"], 168, scale)
    meta["case118_T168"] = dict(sizes=r.sizes, lifted=list(r.lift(1e-4).keys()) and
                                list(r.lifted_sizes))
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
