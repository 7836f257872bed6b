for V in default notdeg; do
  if [ $V = default ]; then unset SPOLY_LIB; else export SPOLY_LIB=$PWD/variants/$V.so; fi
  timeout 600 python bench.py --config C5 --res 128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c5_$V.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/c5_$V.json').read().strip().splitlines()[-1])
print('$V', 'ms %.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['phase_ms'].items()}, d['counters'], d['roofline']['flop_per_launch'])
"
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5_$V.csv \
    python bench.py --config C5 --res 128 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
