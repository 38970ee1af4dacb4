"""GPU: the multi-rank path of bench.py end to end on the one GPU this pool has
(GN_BENCH_ONE_GPU=1: every rank on cuda:0, a gloo group, the ramp halo staged through host
memory, so no kernel waits on another process's kernel).  It checks the plumbing the driver's
scaling runs use -- period shards per rank, the max-over-ranks timing, the nnz all-reduce,
the JSON line from rank 0 -- not its timings.  The peer-memory halo itself is covered by
tests/test_halo.py."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("strong,ranks", [(False, 3), (True, 2)])
def test_bench_multirank_one_gpu(gpu, strong, ranks):
    """weak scaling over three ranks (the middle one has both halo neighbours), strong over two"""
    periods = 24 if not strong else 48
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(ranks), "--master-addr", "127.0.0.1", "--master-port", str(29530 + int(strong)),
           str(ROOT / "bench.py"), "--gpus", str(ranks), "--steps", "4", "--warmup", "3",
           "--config", "case1354pegase", "--periods", str(periods), "--e2e-steps", "2",
           "--no-ipm-ops", "--no-trial", "--traffic-json", ""]
    if strong:
        cmd.append("--strong")
    env = dict(os.environ, GN_BENCH_ONE_GPU="1")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == ranks and d["value"] > 0 and d["ms_per_step"] > 0
    c = d["config"]
    assert c["parallelism"] == f"period-shard x{ranks}" and c["halo"].startswith("gloo")
    assert c["periods_total"] == (24 * ranks if not strong else 48)
    assert c["periods_per_gpu"] == 24
    assert d["e2e"]["ms_per_step"] > 0
