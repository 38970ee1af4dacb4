mkdir -p gpurun_out
for c in 0 2 3; do
  GRIDNLP_B200_GRID_CAP=$c python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial > gpurun_out/gc.json 2>gpurun_out/gc.err || tail -3 gpurun_out/gc.err
  python -c "import json; d=json.load(open('gpurun_out/gc.json')); print('cap', $c, round(d['ms_per_step'],4), d['launch'], {k: round(v['ms'],4) for k, v in d['kernels'].items() if k in ('k_fz_line','k_opf_set_jac_fused','k_fz_busr<d3>')})"
done
