# A/B of library variants: bench C2 phases + output hash per variant (variants/*.so; default = in-tree build)
for v in default $(cd variants && ls *.so 2>/dev/null | sed 's/\.so$//'); do
  if [ "$v" = default ]; then unset SPOLY_LIB; else export SPOLY_LIB=$PWD/variants/$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ab_$v.json 2>/dev/null
  python variants/hash.py ${HASH_CFG:-C2} >> gpurun_out/ab_hash.txt 2>/dev/null
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
ph = {k: round(x["ms"], 4) for k, x in d["roofline"]["phases"].items()}
print(v, "ms/step %.4f" % d["ms_per_step"], d["phase_ms"], ph, flush=True)
PY
done
