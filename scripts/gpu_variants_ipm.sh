# IPM vector-op kernel times per library variant under build/variants/
LIB=paper_2405_14032_b200/libgridnlp_b200.so
cp $LIB /tmp/lib_default.so
for v in build/variants/*/; do
  n=$(basename $v); cp $v/libgridnlp_b200.so $LIB
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-trial --traffic-json '' > gpurun_out/vi.json 2>gpurun_out/vi_$n.err || tail -3 gpurun_out/vi_$n.err
  python -c "import json; d=json.load(open('gpurun_out/vi.json'))['ipm_vector_ops']; print('$n', round(d['ms'],4), round(d['frac'],3), d['kernels_ms'])"
done
cp /tmp/lib_default.so $LIB
