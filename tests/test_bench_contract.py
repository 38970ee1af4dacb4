"""CPU: the bench.py contract that runs without a GPU -- the reference arm's JSON line
(the reference's own CPU path from oracle/_ref on a bounded sample), rank > 0 of a
torchrun launch exiting silently, and our arm failing loudly (non-zero exit) when there
is no CUDA device instead of falling back to a CPU path."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SMALL = ["--config", "case1354pegase", "--periods", "24", "--steps", "2", "--warmup", "1"]


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line():
    from oracle import bindings as B
    if not B.ref_available():
        pytest.skip("oracle/_ref not built")
    r = _run(["--impl", "reference", *SMALL])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "nnz/s" and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    c = d["cpu_baseline"]
    assert c["kind"] == "reference" and c["cores"] >= 1 and c["value"] == d["value"]
    assert "case1354pegase" in c["sample"] or "case1354pegase" in d["config"]["workload"]
    assert d["e2e"] == {"value": d["value"], "unit": "nnz/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    # the reference arm runs the reference only: same configuration as our arm, and no
    # code of this repository's CUDA library mapped into the process
    assert c["same_config"] is True and c["cpu_model"]
    assert not any("libgridnlp_b200" in x for x in d["libraries_loaded"]), d["libraries_loaded"]
    assert any("libgridnlp_ref" in x for x in d["libraries_loaded"])
    assert c["nnz_per_unit"] == {"J": 884552, "H": 1948020, "M": 1083508}


def test_m_nnz_affine_in_periods():
    """The reference arm extrapolates M nnz affinely in T from two period windows (every
    coupling but ramp is per period): exact against the C restatement's full KKT."""
    from oracle import bindings as B
    from paper_2405_14032_b200.network import synthetic_case
    raw = synthetic_case(50, 80, 12, 40, seed=3, parallel_lines=3, shared_gens=2)
    net = raw.network()
    m = {}
    for T in (2, 5, 11):
        Mo = B.OracleModel(net, T, B.np.ones((T, net.n_load)))
        Mo.lift(1e-4)
        m[T] = Mo.kkt().m_nnz
    slope = (m[5] - m[2]) / 3
    assert m[11] == m[5] + slope * 6


def test_reference_arm_other_ranks_exit_silently():
    r = _run(["--impl", "reference", *SMALL], env={"WORLD_SIZE": "2", "RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_our_arm_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run(SMALL)
    assert r.returncode != 0
    assert r.stdout.strip() == ""  # no JSON line from a CPU fallback
