python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | grep -v "^\s*$" | tail -8
for s in 1 2; do python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --streams $s > gpurun_out/bq_$s.json 2> gpurun_out/bq_$s.err || tail -5 gpurun_out/bq_$s.err; done
python - <<'PY'
import json
for s in (1,2):
    d=json.load(open("gpurun_out/bq_%d.json"%s)); print(s, round(d["ms_per_step"],4), {k: round(v,3) for k,v in d.get("stages_ms").items()}, round(d["unit_roofline"]["frac"],3))
    print({k:round(v["ms"],4) for k,v in list(d["kernels"].items())[:16]})
PY
