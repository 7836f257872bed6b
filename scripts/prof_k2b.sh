# k2_build source-correlated stall profile (cuda,sass), a C4 launch list of the current build, cull-level sweep
set -x
T=gpurun_out/${TAG:-pk3}
mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:k2_build -c 1 --launch-skip 2 \
  -o /tmp/kb -f python bench.py --config C4 --res 32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/kb.log 2>&1
$NCU -i /tmp/kb.ncu-rep --page source --csv --print-source cuda,sass > $T/kb.cudasass.csv 2>/dev/null
$NCU -i /tmp/kb.ncu-rep --page details > $T/kb.details.txt 2>/dev/null
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_C4.csv \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/launches_C4.log 2>&1
for L in 2 4 5; do
  timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --cull-levels $L > $T/lv$L.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$T/lv$L.json').read().strip().splitlines()[-1])
print('levels $L', 'ms %.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['phase_ms'].items()}, d['counters']['n_admissible'], d['pairs_per_step_per_gpu'])
"
done
ls -la $T
