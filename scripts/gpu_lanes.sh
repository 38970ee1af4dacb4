# bus-class lanes of the fused KKT (GRIDNLP_B200_BUS_LANES) per config; "" = the default rule
mkdir -p gpurun_out
for cfg in "case1354pegase 24" "case9241pegase 48" "synthetic30k 96"; do
  set -- $cfg
  for ln in "" 1 2 4 8; do
    GRIDNLP_B200_BUS_LANES=$ln python bench.py --config $1 --periods $2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --traffic-json '' > gpurun_out/ln.json 2>gpurun_out/ln.err || tail -3 gpurun_out/ln.err
    python -c "import json; d=json.load(open('gpurun_out/ln.json')); print('$1', 'lanes=$ln', round(d['ms_per_step'],4), d['launch'], d['clocks']['sm_mhz'])"
  done
done
