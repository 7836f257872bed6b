# ncu captures of the one-bounce kernels at the C2 bench config (one GPU), then the launch list of a short run
set -x
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:"${KREGEX:-k1_phase1|k1_path_fast}" -c ${KCOUNT:-2} \
  -o gpurun_out/${TAG:-p}_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/${TAG:-p}_full.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-p}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/${TAG:-p}_launches.log 2>&1
ls -la gpurun_out/
