# usage: bash scripts/gpu_prof1.sh <tag> <kernel regex> [bench args...]
# plain run first (must exit 0), then one ncu --set full capture (one launch) of the kernel,
# eager on one stream so it runs alone
tag=$1; re=$2; shift 2
mkdir -p gpurun_out
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --no-seam --graph 0 --streams 1 $@"
$C > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$tag.log; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$re" -s 1 -c 1 -o gpurun_out/prof_$tag $C > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"
