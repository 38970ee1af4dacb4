# A/B: the default build against each build/variants/* (GRIDNLP_B200_LIB), alternating, N rounds
# usage: bash scripts/gpu_ab.sh [rounds] [bench args]
R=${1:-2}; shift
mkdir -p gpurun_out
B="python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --no-seam --traffic-json ''"
show() { python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); k=d['kernels']; print('$1', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], {x: round(k[x]['ms'],4) for x in list(k)[:7]})"; }
for i in $(seq $R); do
  $B "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err && show default || tail -3 gpurun_out/ab.err
  for v in build/variants/*/; do
    n=$(basename $v)
    GRIDNLP_B200_LIB=$PWD/$v/libgridnlp_b200.so $B "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err && show $n || tail -3 gpurun_out/ab.err
  done
done
