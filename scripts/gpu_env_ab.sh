# paired A/B of an environment knob on bench.py: bash scripts/gpu_env_ab.sh VAR "v1 v2" rounds [bench args]
var=$1; vals=$2; R=${3:-3}; shift 3
mkdir -p gpurun_out
B="python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --no-seam --traffic-json ''"
for i in $(seq $R); do
  for v in $vals; do
    env $var=$v $B "$@" > gpurun_out/eab.json 2>gpurun_out/eab.err || { tail -3 gpurun_out/eab.err; continue; }
    python -c "import json; d=json.load(open('gpurun_out/eab.json')); k=d['kernels']; print('$var=$v', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], {x: round(k[x]['ms'],4) for x in list(k)[:4]})"
  done
done
