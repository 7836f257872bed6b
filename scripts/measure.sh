# Round measurement on one B200: bench lines for every config, launch lists (C2, C4), ncu --set full captures of
# the top one-bounce and two-bounce kernels.  Outputs land in gpurun_out/$TAG/.
set -x
T=gpurun_out/${TAG:-m}
mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $T/smi.txt
timeout 600 python bench.py > $T/bench_C2.json 2> $T/bench_C2.err
for c in C1 C3 C4 C5RR; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $T/bench_$c.json 2> $T/bench_$c.err
done
timeout 900 python bench.py --config C5 --res 128 --steps 3 --warmup 3 > $T/bench_C5.json 2> $T/bench_C5.err
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $T/launches_C2.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_C4.csv \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/launches_C4.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"k1_phase1|k1_path_fast|k_query_cull" -c 4 \
  -o $T/k1_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/k1_full.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"k2_build|k2_scan|k_pair_expand|k_refine_level" -c 6 \
  -o $T/k2_full -f python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $T/k2_full.log 2>&1
ls -la $T
