# Two-bounce re-measurement after the last k2 changes (outputs in gpurun_out/$TAG)
set -x
T=gpurun_out/${TAG:-fk2}
mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
for c in C4 C5RR; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $T/bench_$c.json 2> $T/bench_$c.err
done
timeout 900 python bench.py --config C5 --res 128 --steps 3 --warmup 3 > $T/bench_C5.json 2> $T/bench_C5.err
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_C4.csv \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/launches_C4.log 2>&1
for KS in k2_build:2 k2_scan:1 k_refine_level:2; do
  K=${KS%%:*}; S=${KS##*:}
  $NCU --set full --clock-control none -k regex:"$K" -c 1 --launch-skip $S -o /tmp/$K -f \
    python bench.py --config C4 --res 32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/$K.log 2>&1
  $NCU -i /tmp/$K.ncu-rep --page raw --csv > $T/$K.raw.csv 2>/dev/null
done
timeout 1500 python profiles/run_c5_full.py > $T/c5_full.json 2> $T/c5_full.err
ls -la $T
