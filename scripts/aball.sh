# A/B of library variants over one- and two-bounce configs: output hashes + ms/step and phases
run() {
  timeout 900 python bench.py --config $1 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e $2 > gpurun_out/aball.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/aball.json').read().strip().splitlines()[-1])
print('$1 $2 ${V}', 'ms %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['phase_ms'].items()}, d['pairs_per_step_per_gpu'], round(d['roofline']['frac'],4), flush=True)
"
}
for V in default ${VARIANTS:-$(cd variants && ls *.so 2>/dev/null | sed 's/\.so$//')}; do
  if [ $V = default ]; then unset SPOLY_LIB; else export SPOLY_LIB=$PWD/variants/$V.so; fi
  python variants/hash.py C2
  python variants/hash.py C3
  python variants/hash.py C4
  run C2 "" 10; run C3 "" 5; run C4 "" 3; run C5 "--res 128" 3
done
