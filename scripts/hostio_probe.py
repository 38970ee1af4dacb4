"""Host-mode transfer rates of the C-ABI (GN_MEM_HOST, pageable numpy buffers) at the bench
workload: eval_hess (1.4 GB back), eval_jac, and KKT set_jacobian / assemble / values."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
from helpers import interior_point, row_weights, sigmas  # noqa: E402
from paper_2405_14032_b200.network import config_case  # noqa: E402
from paper_2405_14032_b200.opf import CondensedKkt, OpfNlp, load_profile  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 96
net = config_case("synthetic30k").network()
nlp = OpfNlp(net, T, load_profile(net.n_load, T))
xl, xu, xs, _, _ = nlp.bounds()
x = interior_point(xl, xu, xs, 1)
w = row_weights(nlp.n_cons(), 2)
H = np.empty(nlp.sizes.hess_nnz)
J = np.empty(nlp.sizes.jac_nnz)
H.fill(0.0)
J.fill(0.0)


def timed(fn, nbytes, what, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    t = min(ts)
    print(f"{what:40s} {t * 1e3:8.1f} ms  {nbytes / t / 1e9:6.1f} GB/s")


timed(lambda: nlp.eval_hess(x, w, 1.0, out=H), H.nbytes + x.nbytes + w.nbytes, "eval_hess host (x, w in; H out)")
timed(lambda: nlp.eval_jac(x, out=J), J.nbytes + x.nbytes, "eval_jac host (x in; J out)")
nlp.lift(1e-4)
K = CondensedKkt(nlp=nlp)
L = nlp.lifted_structure()
jl, hl = J[L["jac_pick"]], H[L["hess_pick"]]
sx, ss = sigmas(nlp.sizes.n_free, nlp.n_cons(), 3)
timed(lambda: K.set_jacobian(jl), jl.nbytes, "set_jacobian host (J_l in)")
timed(lambda: K.assemble(hl, sx, ss, 1e-4, 1e-8), hl.nbytes + sx.nbytes + ss.nbytes, "assemble host (H_l, sigma in)")
a, m = np.empty(K.a_nnz), np.empty(K.m_nnz)
timed(lambda: K.values(a, m), a.nbytes + m.nbytes, "values host (A, M out)")
