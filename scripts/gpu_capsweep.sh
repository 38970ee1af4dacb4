mkdir -p gpurun_out
run() {  # SETJAC LINE BUS
  GRIDNLP_B200_GRID_CAP=2 GRIDNLP_B200_GRID_CAP_SETJAC=$1 GRIDNLP_B200_GRID_CAP_LINE=$2 GRIDNLP_B200_GRID_CAP_BUS=$3 \
    python bench.py --steps 150 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --no-dropin > gpurun_out/cs.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/cs.json')); print('sj', $1, 'line', $2, 'bus', $3, round(d['ms_per_step'],4))"
}
for rep in 1 2; do
  run 2 2 2; run 0 2 2; run 3 2 2; run 4 2 2; run 2 0 2; run 2 3 2; run 2 2 0; run 2 2 3; run 2 2 4
done
