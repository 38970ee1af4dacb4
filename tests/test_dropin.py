"""GPU, end to end: the UNMODIFIED reference interior-point driver
(ipm::solve_nlp, solver.hpp:469) running on the B200 path through the
reference's own seams — CudaOpfNlp (NlpProblem, nlp.hpp:15-39) and the shadowed
CondensedKkt (condensed.hpp:27-185).  Iteration count and objective must match
the reference's own solves (tests/golden/meta.json, produced by oracle/_ref) to
1e-6 relative at tol 1e-4 (BASELINE.json north_star)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from helpers import golden_meta, golden_network
from paper_2405_14032_b200.opf import load_profile

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
DROPIN = ROOT / "oracle" / "_ref" / "ipm_dropin"


def write_bin(path, net, T, scale):
    with open(path, "wb") as f:
        np.array([net.n_bus, net.n_line, net.n_gen, net.n_load, net.reference_bus, T],
                 np.int32).tofile(f)
        np.array([net.base_mva], np.float64).tofile(f)
        for k in ("bus_vmin", "bus_vmax", "vm_start", "va_start"):
            getattr(net, k).tofile(f)
        net.line_from.tofile(f)
        net.line_to.tofile(f)
        for k in ("line_g", "line_b", "line_smax", "line_amin", "line_amax"):
            getattr(net, k).tofile(f)
        net.gen_bus.tofile(f)
        for k in ("gen_pmin", "gen_pmax", "gen_qmin", "gen_qmax", "gen_ramp", "gen_c2", "gen_c1",
                  "gen_c0", "gen_pstart", "gen_qstart", "gen_qstart"):
            getattr(net, k).tofile(f)
        net.load_bus.tofile(f)
        net.load_p.tofile(f)
        net.load_q.tofile(f)
        np.ascontiguousarray(scale, np.float64).tofile(f)


@pytest.mark.parametrize("key", ["case9_T1", "case30_T30_r30", "case118_T24"])
@pytest.mark.parametrize("nlp", ["cuda", "ref"])
def test_reference_ipm_on_b200_path(gpu, tmp_path, key, nlp):
    if not DROPIN.exists():
        pytest.skip("oracle/_ref/ipm_dropin not built (needs /root/reference at build time)")
    g = golden_meta()["solves"][key]
    net = golden_network(g["case"])
    scale = load_profile(net.n_load, g["periods"], g["resolution"], seed=1)
    path = tmp_path / "net.bin"
    write_bin(path, net, g["periods"], scale)
    out = subprocess.run([str(DROPIN), str(path), nlp], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["status"] == "solved"
    assert r["iterations"] == g["iterations"], (r, g)
    assert abs(r["objective"] - g["objective"]) <= 1e-6 * abs(g["objective"]), (r, g)
