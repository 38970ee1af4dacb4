# IPM vector-op kernel times per library variant under build/variants/
for v in build/variants/*/; do
  n=$(basename $v)
  export GRIDNLP_B200_LIB=$PWD/$v/libgridnlp_b200.so
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-trial --traffic-json '' > gpurun_out/vi.json 2>gpurun_out/vi_$n.err || tail -3 gpurun_out/vi_$n.err
  python -c "import json; d=json.load(open('gpurun_out/vi.json'))['ipm_vector_ops']; print('$n', round(d['ms'],4), round(d['frac'],3), d['kernels_ms'])"
done
