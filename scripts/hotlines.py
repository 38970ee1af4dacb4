"""Top CUDA source lines of one kernel in an ncu report by warp-stall samples
(ncu --page source --print-source cuda,sass; the library is built with -lineinfo).
usage: python scripts/hotlines.py <report.ncu-rep> [n] [function-name substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines, path, hdr, take = [], "", None, True
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r and r[0] == "Function Name":
        take = want is None or want in r[1]
    elif not take:
        continue
    elif r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
    elif hdr and r and r[0] and r[0] != "Function Name":
        try:
            s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            ins = int(r[hdr["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        lines.append((s, ins, f"{path}:{r[0]}", r[1].strip()[:90]))
tot = sum(x[0] for x in lines) or 1
toti = sum(x[1] for x in lines) or 1
print(f"{tot} stall samples, {toti} warp instructions")
for s, ins, loc, src in sorted(lines, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  {100 * ins / toti:5.1f}%i  {loc:28s} {src}")
