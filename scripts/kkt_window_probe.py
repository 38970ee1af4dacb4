"""How well does the reference arm's CondensedKkt extrapolation hold?  Times the reference's
own CondensedKkt::set_jacobian + assemble (oracle/_ref) on period windows of a BASELINE
network and prints ns per J_l entry / per assembly contribution for each window length.
usage: python scripts/kkt_window_probe.py [config] [T1 T2 ...]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import bench  # noqa: E402
from oracle import bindings as B  # noqa: E402
from paper_2405_14032_b200.network import config_case  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "synthetic30k"
wins = [int(a) for a in sys.argv[2:]] or [2, 8, 24]
raw = config_case(config, seed=1)
text = raw.to_matpower()
scale = B.ref_load_profile(text, max(wins))
for Tw in wins:
    t0 = time.perf_counter()
    W = B.RefModel(text, Tw, scale[:Tw])
    lw = W.lift(1e-4)
    nlw, mw, njw, nhw = W.lifted_sizes
    Pw = bench._pairs(lw["jac_rows"], mw)
    dims = W.kkt_create()
    ctor_s = time.perf_counter() - t0
    xw, ww, sxw, ssw = bench.inputs(W.bounds()[:3], mw, nlw)
    xf = np.ascontiguousarray(xw[lw["free_to_full"]])
    jw, hw = np.empty(njw), np.empty(nhw)
    assert W.L.gnr_lifted_eval_jac(W.h, B._f(xf), B._f(jw))
    assert W.L.gnr_lifted_eval_hess(W.h, B._f(xf), B._f(ww), 1.0, B._f(hw))
    sj, sa = [], []
    for _ in range(3):
        a = time.perf_counter()
        W.kkt_set_jacobian(jw)
        b = time.perf_counter()
        W.kkt_assemble(hw, sxw, ssw, 1e-4, 1e-8 * 0.1 ** 0.25)
        sj.append(b - a)
        sa.append(time.perf_counter() - b)
    print(json.dumps(dict(config=config, periods=Tw, setup_s=round(ctor_s, 1),
                          set_jacobian_ms=1e3 * float(np.median(sj)),
                          assemble_ms=1e3 * float(np.median(sa)),
                          ns_per_jac=1e9 * float(np.median(sj)) / njw,
                          ns_per_contribution=1e9 * float(np.median(sa)) / (nhw + Pw + nlw))),
          flush=True)
    del W
