# KKT concurrency sweep: set_jacobian forked or serial x grid cap, two configs
mkdir -p gpurun_out
for cfg in "case9241pegase 48" "synthetic30k 96"; do
  set -- $cfg
  for sj in 1 0; do
    for cap in 2 1 3 0; do
      GRIDNLP_B200_SETJAC_FORK=$sj python bench.py --config $1 --periods $2 --grid-cap $cap --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --traffic-json '' > gpurun_out/ks.json 2>gpurun_out/ks.err || tail -3 gpurun_out/ks.err
      python -c "import json; d=json.load(open('gpurun_out/ks.json')); print('$1', 'setjac_fork=$sj cap=$cap', round(d['ms_per_step'],4), d['launch'], d['clocks']['sm_mhz'])"
    done
  done
done
