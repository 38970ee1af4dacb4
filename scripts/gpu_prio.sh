mkdir -p gpurun_out
for cfg in "0 -1" "-1 0" "0 0" "-1 -1"; do
  set -- $cfg
  GN_CB_PRIORITY=$1 GN_KKT_PRIORITY=$2 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops > gpurun_out/prio.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/prio.json')); print('cb', $1, 'kkt', $2, round(d['ms_per_step'],4), d['launch'])"
done
