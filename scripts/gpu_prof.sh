# usage: bash scripts/gpu_prof.sh <tag> <kernel regex> [count]
# plain run first (must exit 0), then one ncu --set full capture of the matching kernels
tag=$1; re=$2; cnt=${3:-4}
mkdir -p gpurun_out
C="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --streams 1"
$C > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$tag.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$re" -s ${4:-40} -c $cnt -o gpurun_out/prof_$tag $C > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"
