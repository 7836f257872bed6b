for V in default skipb; do
  if [ $V = default ]; then unset SPOLY_LIB; else export SPOLY_LIB=$PWD/variants/$V.so; fi
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k2_build --csv --log-file gpurun_out/skipb_$V.csv \
    python bench.py --config C4 --res 64 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python profiles/launch_shares.py gpurun_out/skipb_$V.csv 3
done
