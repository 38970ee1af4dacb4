# callback issue order vs the KKT stream: step time per order (graph mode and eager)
mkdir -p gpurun_out
for o in "f,grad,g,jac,hess" "hess,jac,g,grad,f" "hess,f,grad,g,jac" "jac,hess,f,grad,g" "g,hess,jac,f,grad"; do
  GN_CB_ORDER=$o python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial > gpurun_out/ord.json 2>gpurun_out/ord.err || tail -3 gpurun_out/ord.err
  python -c "import json; d=json.load(open('gpurun_out/ord.json')); print('$o', round(d['ms_per_step'],4), d['launch'], d['clocks']['sm_mhz'])"
done
