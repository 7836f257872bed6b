export SPOLY_PARITY_LOG=gpurun_out/parity10.jsonl
timeout 1200 python -m pytest tests -m gpu -q -rf --durations=5 > gpurun_out/gputest10.log 2>&1; echo PYTEST_EXIT $?
run() {
  timeout 600 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $2 > gpurun_out/k2ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/k2ab.json').read().strip().splitlines()[-1])
print('$1 $2', 'ms %.1f'%d['ms_per_step'], {k:round(v,1) for k,v in d['phase_ms'].items()}, d['counters']['n_admissible'], d['pairs_per_step_per_gpu'], d['counters']['n_pairs_coarse'], d['counters']['n_cull_tests'])
"
}
run C4 ""; run "C5 --res 128" "--k2-tiles 0"; run "C5 --res 128" ""; run C5RR ""
