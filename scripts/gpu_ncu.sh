tag=$1
mkdir -p gpurun_out
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --no-seam --graph 0 --streams 1"
$C > gpurun_out/plain_launch_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_$tag.csv $C > gpurun_out/ncu_launch_$tag.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_eval|k_fz_line|k_fz_busr|k_fz_bus3|k_opf_set_jac_fused|k_fz_dvec|k_bus|k_fz_gen" -s 40 -c 16 -o gpurun_out/full_$tag $C > gpurun_out/ncu_full_$tag.log 2>&1
echo "full capture rc=$?"
