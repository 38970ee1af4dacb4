# Round-end evidence: GPU tests, default bench (both arms), ncu launch list, one full capture.
# usage: bash scripts/gpu_round.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || { echo "bench failed"; tail -5 gpurun_out/bench_$tag.err; exit 1; }
python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err || echo "reference arm failed"
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --no-seam --graph 0 --streams 1"
$C > gpurun_out/plain_launch_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv $C > gpurun_out/ncu_launch_$tag.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_eval|k_fz_line|k_fz_busr|k_fz_bus3|k_opf_set_jac_fused|k_fz_dvec|k_bus|k_fz_gen" -s 40 -c 16 -o gpurun_out/full_$tag $C > gpurun_out/ncu_full_$tag.log 2>&1
echo "full capture rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_$tag.json')); print({k: d[k] for k in ('value','ms_per_step','launch','roofline','unit_roofline','clocks','gpu_launches','line_search_trial','ipm_vector_ops')}); print('e2e', d['e2e']); print('cpu', d['cpu_baseline'])
d=json.load(open('gpurun_out/bench_ref_$tag.json')); print('ref', d.get('value'), d.get('unit'), d.get('cpu_baseline'))"
