run() {
  timeout 600 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $2 > gpurun_out/k2ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/k2ab.json').read().strip().splitlines()[-1])
print('$1 $2 ${SPOLY_LIB}', 'ms %.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['phase_ms'].items()}, d['counters']['n_admissible'], d['pairs_per_step_per_gpu'], d['roofline']['frac'])
"
}
for v in default refl0 refsph; do
  if [ $v = default ]; then unset SPOLY_LIB; else export SPOLY_LIB=$PWD/variants/$v.so; fi
  run C4 ""; run "C5 --res 128" ""
done
