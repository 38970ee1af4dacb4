# usage: bash scripts/gpu_env_sweep.sh VAR "v1 v2 ..." kernel_regex
var=$1; vals=$2; kre=$3
mkdir -p gpurun_out
for v in $vals; do
  env $var=$v python bench.py --steps 10 --warmup 4 --no-e2e --no-cpu-baseline --streams 1 > gpurun_out/sw_$v.json 2> gpurun_out/sw_$v.err || tail -3 gpurun_out/sw_$v.err
  python - "$v" "$kre" <<'PY'
import json, re, sys
v, kre = sys.argv[1], sys.argv[2]
d = json.load(open("gpurun_out/sw_%s.json" % v))
ks = {k: round(x["ms"], 4) for k, x in d["kernels"].items() if re.search(kre, k)}
print(v, round(d["ms_per_step"], 4), ks)
PY
done
