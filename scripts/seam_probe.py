"""Time the drop-in seams (oracle/_ref/seam_bench) at a BASELINE configuration, both
LiftedProblem modes: python scripts/seam_probe.py [config] [periods] [units]."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else bench.CONFIG
periods = int(sys.argv[2]) if len(sys.argv) > 2 else bench.PERIODS_PER_RANK
units = int(sys.argv[3]) if len(sys.argv) > 3 else 3
raw, net, scale = bench.build_workload(0, 1, periods, config)
r = bench.dropin_seam(raw, net, scale, units=units)
print(json.dumps(dict(config=config, periods=periods, **(r or {"error": "seam_bench missing"}))))
