# A/B of library variants on the two-bounce configs: ms/step + phase split + output hash (C4 subset) per variant
run() {
  timeout 900 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $2 > gpurun_out/k2ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/k2ab.json').read().strip().splitlines()[-1])
print('$1 $2 ${V}', 'ms %.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['phase_ms'].items()}, d['counters']['n_admissible'], d['pairs_per_step_per_gpu'], round(d['roofline']['frac'],4), flush=True)
"
}
for V in default ${VARIANTS:-$(cd variants && ls *.so 2>/dev/null | sed 's/\.so$//')}; do
  if [ $V = default ]; then unset SPOLY_LIB; else export SPOLY_LIB=$PWD/variants/$V.so; fi
  python variants/hash.py C4
  python variants/hash.py C5RR
  run C4 ""; run C5 "--res 128"
done
