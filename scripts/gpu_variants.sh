# bench every library variant under build/variants/ (scripts/build_variant.py) on the default
# workload; each variant is loaded through GRIDNLP_B200_LIB (the in-tree library is never overwritten).  usage: bash scripts/gpu_variants.sh [bench args]
mkdir -p gpurun_out
for v in build/variants/*/; do
  n=$(basename $v)
  export GRIDNLP_B200_LIB=$PWD/$v/libgridnlp_b200.so
  python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --traffic-json '' "$@" > gpurun_out/var.json 2>gpurun_out/var_$n.err || tail -3 gpurun_out/var_$n.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); k=d['kernels']; print('$n', '$(cat $v/defines.txt)', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], {x: round(k[x]['ms'],4) for x in list(k)[:8]})"
done
