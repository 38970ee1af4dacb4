for i in 1 2; do for v in build/variants/*/; do
  n=$(basename $v)
  export GRIDNLP_B200_LIB=$PWD/$v/libgridnlp_b200.so
  python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --traffic-json '' > gpurun_out/vt.json 2>gpurun_out/vt_$n.err || tail -3 gpurun_out/vt_$n.err
  python -c "import json; d=json.load(open('gpurun_out/vt.json')); print('$n', round(d['ms_per_step'],4), d['line_search_trial']['ms'], d['kernels']['k_eval<G>']['ms'])"
done; done
