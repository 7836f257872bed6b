# Round-2 final measurement on one B200 (outputs in gpurun_out/$TAG): bench lines, reference arm, launch lists,
# ncu --set full summaries (raw CSV + details, the .ncu-rep files stay on the box), the full C5 sweep.
set -x
T=gpurun_out/${TAG:-fin}
mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $T/smi.txt
timeout 600 python bench.py > $T/bench_C2.json 2> $T/bench_C2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $T/bench_ref.json 2> $T/bench_ref.err
for c in C1 C3 C4 C5RR; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $T/bench_$c.json 2> $T/bench_$c.err
done
timeout 900 python bench.py --config C5 --res 128 --steps 3 --warmup 3 > $T/bench_C5.json 2> $T/bench_C5.err
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $T/launches_C2.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_C4.csv \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/launches_C4.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:"k1_phase1|k1_path_fast|k_tile_query_cull|k_tile_cull|k1_roots_deep" -c 12 \
  -o /tmp/k1f -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/k1_full.log 2>&1
$NCU -i /tmp/k1f.ncu-rep --page raw --csv > $T/k1_full.raw.csv 2>/dev/null
$NCU -i /tmp/k1f.ncu-rep --page details > $T/k1_full.details.txt 2>/dev/null
for KS in k2_build:2 k2_scan:1 k_refine_level:2; do
  K=${KS%%:*}; S=${KS##*:}
  $NCU --set full --clock-control none -k regex:"$K" -c 1 --launch-skip $S -o /tmp/$K -f \
    python bench.py --config C4 --res 32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/$K.log 2>&1
  $NCU -i /tmp/$K.ncu-rep --page raw --csv > $T/$K.raw.csv 2>/dev/null
  $NCU -i /tmp/$K.ncu-rep --page details > $T/$K.details.txt 2>/dev/null
done
timeout 1500 python profiles/run_c5_full.py > $T/c5_full.json 2> $T/c5_full.err
ls -la $T
