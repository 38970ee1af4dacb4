"""Summarise ncu outputs into the small text files committed under profiles/.

  python profiles/summarize.py launches <launches.csv> <out.md>
      per-kernel launch count, total / mean device time and share of the
      timed steps (from `ncu --metrics gpu__time_duration.sum --csv`)
  python profiles/summarize.py full <report.ncu-rep> <out.md> [traffic.json]
      key metrics of every profiled kernel of an `ncu --set full` capture
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__registers_per_thread", "registers"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cycles/inst"),
]


def short(name: str) -> str:
    return name.split("(")[0].replace("void ", "").strip()


MODES = {"0": "F", "1": "GRAD", "2": "G", "3": "J", "4": "H", "5": "FG"}


def pretty(name: str) -> str:
    """gnb::k_eval<4> -> k_eval<H>; value-mode fused kernels <0> -> plain name."""
    n = name.replace("gnb::", "")
    for k in ("k_eval", "k_line", "k_gen", "k_thermal", "k_ramp"):
        if n.startswith(k + "<") and n[len(k) + 1:-1] in MODES:
            return f"{k}<{MODES[n[len(k) + 1:-1]]}>"
    import re
    mm = re.fullmatch(r"k_fz_busr<(\d+), 0>", n)
    if mm:
        return f"k_fz_busr<d{mm.group(1)}>"
    for k in ("k_fz_bus3", "k_fz_line", "k_fz_gen", "k_opf_assemble"):
        if n == k + "<0>" or n.startswith(k + "<0, "):  # (k_fz_line<STRUCT, FLAT>)
            return k
        if n == k + "<1>" or n.startswith(k + "<1, "):
            return k + " (structure check)"
    return n


def launches(path: str, out: str):
    """Per-step kernel table of an ncu launch list of `bench.py --steps K --warmup W`:
    kernels launched a multiple of S times (S = warm-up + timed + profiled steps,
    the most common launch count) are the step's kernels; the rest ran once at setup."""
    from collections import Counter
    text = open(path).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = [r for r in csv.DictReader(text[start:]) if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)
        agg.setdefault(short(r["Kernel Name"]), []).append(us)
    counts = Counter(len(v) for k, v in agg.items() if k.startswith("gnb::"))
    # steps in the capture = launches of a once-per-step kernel (the Hessian callback)
    hk = next((k for k in ("gnb::k_eval<4>", "gnb::k_line<4>") if k in agg), None)
    S = len(agg[hk]) if hk else max(counts, key=lambda c: (counts[c], c))
    step = {k: v for k, v in agg.items() if len(v) % S == 0 and k.startswith("gnb::")}
    setup = {k: v for k, v in agg.items() if k not in step}
    tot = sum(sum(v) for v in step.values()) / S
    lines = [f"Per-step kernels ({S} steps in the capture: warm-up + timed + profiled; "
             "ncu serialises launches and runs them cold, so the SHARE column is the "
             "comparable figure, not the absolute time).", "",
             "| kernel | launches / step | us / step | us / launch | share of step |",
             "|---|---:|---:|---:|---:|"]
    for k, v in sorted(step.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{pretty(k)}` | {len(v) // S} | {sum(v) / S:.1f} | {sum(v) / len(v):.2f} "
                     f"| {sum(v) / S / tot:.1%} |")
    lines.append(f"\n{tot / 1000:.3f} ms of kernel time per step.  Setup (once per context / KKT "
                 f"object, not in the step): {len(setup)} kernels, "
                 f"{sum(sum(v) for v in setup.values()) / 1000:.3f} ms.")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep: str, out: str, traffic_json: str | None = None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    lines = ["| kernel | " + " | ".join(lbl for _, lbl in KEYS) + " |",
             "|---|" + "---:|" * len(KEYS)]
    traffic = {}
    seen: dict = {}
    for r in rows[2:]:
        name = pretty(short(r[head.index("Kernel Name")]))
        seen[name] = seen.get(name, 0) + 1
        first = seen[name] == 1
        if not first:  # the capture window reached into the next step: table only
            name = f"{name} #{seen[name]}"
        cells = []
        for key, _ in KEYS:
            try:
                i = head.index(key)
                cells.append(f"{r[i]} {units[i]}".strip())
            except ValueError:
                cells.append("-")
        lines.append(f"| `{name}` | " + " | ".join(cells) + " |")
        try:
            rd = float(r[head.index("dram__bytes_read.sum")]) * _scale(units[head.index("dram__bytes_read.sum")])
            wr = float(r[head.index("dram__bytes_write.sum")]) * _scale(units[head.index("dram__bytes_write.sum")])
            if first:
                traffic[name] = rd + wr
        except (ValueError, IndexError):
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json:
        json.dump(traffic, open(traffic_json, "w"), indent=1)


def _scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
