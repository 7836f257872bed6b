VARIANTS="notdeg unk" bash scripts/abk2.sh > gpurun_out/abk2_7.log 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4_r2e.csv \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_C4_r2e.log 2>&1
export SPOLY_LIB=$PWD/variants/notdeg.so
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4_r2e_notdeg.csv \
  python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_C4_r2e_nd.log 2>&1
