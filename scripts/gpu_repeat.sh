# the default bench step, repeated: run-to-run spread of the headline number on one box
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
  python bench.py --no-e2e --no-cpu-baseline --no-ipm-ops --no-trial --steps 200 --warmup 5 > gpurun_out/rep_$i.json 2>gpurun_out/rep_$i.err || tail -3 gpurun_out/rep_$i.err
  python -c "import json; d=json.load(open('gpurun_out/rep_$i.json')); print($i, round(d['ms_per_step'],4), round(d['value']/1e11,4), round(d['unit_roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
