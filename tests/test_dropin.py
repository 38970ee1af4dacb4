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


from oracle.bindings import write_network_bin as write_bin  # noqa: E402


# SURVEY §8(c) goldens: case118 x 168 is the survey's 40-iteration solve (objective
# 10578502.183425546); case1354s x 24 is BASELINE configs[1]'s size;
# synthloop x 4 carries two self-loop lines (the OPF-specialised KKT declines those
# networks, so the shim's CondensedKkt runs the generic kernels on our callbacks)
# synthinf x 3 is overloaded: the reference enters feasibility restoration (the
# restoration problem wraps the same LiftedProblem, restoration.hpp:24) and ends infeasible
KEYS = ["case9_T1", "case30_T30_r30", "case118_T24", "case118_T168", "case1354s_T24",
        "synthloop_T4", "synthinf_T3"]
STATUS = ["solved", "max_iterations", "infeasible", "unrecoverable"]  # solver.hpp:20-25
GENERIC_ONLY = {"synthloop_T4"}


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("nlp", ["cuda", "ref"])
def test_reference_ipm_on_b200_path(gpu, tmp_path, key, nlp):
    """nlp = cuda: CudaOpfNlp + the shim CondensedKkt (recognised as the OPF problem:
    specialised assembly); nlp = ref: the reference's PatternNlp callbacks + the shim
    CondensedKkt on the generic contributor-list kernels."""
    if not DROPIN.exists():
        pytest.skip("oracle/_ref/ipm_dropin not built (needs /root/reference at build time)")
    g = golden_meta()["solves"][key]
    net = golden_network(g["case"])
    scale = load_profile(net.n_load, g["periods"], g["resolution"], seed=1)
    path = tmp_path / "net.bin"
    write_bin(path, net, g["periods"], scale)
    out = subprocess.run([str(DROPIN), str(path), nlp], capture_output=True, text=True,
                         timeout=1200)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["status"] == STATUS[int(g["status"])], (r, g)
    assert r["iterations"] == g["iterations"], (r, g)
    assert r["restorations"] == g["restorations"], (r, g)
    # the seam reached the specialised kernels exactly when the callbacks are ours
    specialised = nlp == "cuda" and key not in GENERIC_ONLY
    # (a feasibility restoration builds its own KKT on the restoration problem's structure:
    # generic, solver.hpp:413-419)
    assert (r["kkt_specialised"] >= 1 and r["kkt_generic"] == r["restorations"]) \
        if specialised else (r["kkt_specialised"] == 0 and r["kkt_generic"] >= 1), r
    # the shim LiftedProblem ran on the device exactly for our callbacks (the restoration
    # problem and PatternNlp keep the reference's own host class)
    assert (r["lifted_device"] >= 1) if nlp == "cuda" else (r["lifted_device"] == 0), r
    assert r["lifted_host"] == r["restorations"] + (0 if nlp == "cuda" else 1), r
    assert abs(r["objective"] - g["objective"]) <= 1e-6 * abs(g["objective"]), (r, g)


LIFTED_CHECK = ROOT / "oracle" / "_ref" / "lifted_check"


@pytest.mark.parametrize("case,periods", [("case118", 24), ("synth", 3), ("case1354s", 4),
                                          ("synthloop", 4)])
def test_lifted_shim_matches_the_reference_class(gpu, tmp_path, case, periods):
    """The shim LiftedProblem over CudaOpfNlp (device mode) against the reference's own
    LiftedProblem over PatternNlp, relative and absolute relaxation: structures, free map,
    boxes, slack boxes and to_full bit for bit; the lifted evaluations within the 1e-12 bar
    (grad bit for bit)."""
    if not LIFTED_CHECK.exists():
        pytest.skip("oracle/_ref/lifted_check not built (needs /root/reference at build time)")
    net = golden_network(case)
    scale = load_profile(net.n_load, periods, 60.0, seed=1)
    path = tmp_path / "net.bin"
    write_bin(path, net, periods, scale)
    out = subprocess.run([str(LIFTED_CHECK), str(path)], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr
    for r in json.loads(out.stdout.strip().splitlines()[-1]):
        assert r["device_mode"] == 1 and r["host_mode"] == 1, r
        assert r["struct_diff"] == 0 and r["boxes_diff"] == 0 and r["to_full_diff"] == 0, r
        assert r["evals_ok"] == 1 and r["grad_diff"] == 0, r
        assert r["max_rel_diff"] <= 1e-12, r
