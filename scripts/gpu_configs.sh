# BASELINE.json configs[1..4] on one B200: one bench line each (configs[0] is the CPU parity
# case, covered by tests/).  The traffic table in profiles/ is for the default workload only.
set -u
mkdir -p gpurun_out
for cfg in "case1354pegase 24" "case9241pegase 48" "case13659pegase 168" "synthetic30k 96"; do
  set -- $cfg
  timeout 900 python bench.py --config $1 --periods $2 --steps 100 --warmup 5 --traffic-json '' \
    > gpurun_out/cfg_$1.json 2> gpurun_out/cfg_$1.err || { echo "FAIL $1"; tail -5 gpurun_out/cfg_$1.err; }
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/cfg_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    c, u = d["cpu_baseline"] or {}, d["unit_roofline"]
    print(f, d["config"]["workload"], "ms %.4f" % d["ms_per_step"], "nnz/s %.3e" % d["value"],
          "unit_frac %.3f" % u["frac"], "dom %s %.3f" % (d["roofline"]["kernel"], d["roofline"]["frac"]),
          "e2e %.3e" % d["e2e"]["value"] if d.get("e2e") else "", "cpu %.3e" % c.get("value", 0),
          d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
