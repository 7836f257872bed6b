# ncu --set full of the top two-bounce kernels (one launch each) at C4 with 1,024 queries; exports the raw metrics,
# the details page and the per-line source page (the .ncu-rep files stay on the box: gpurun copies back <= 64 MiB)
set -x
T=gpurun_out/${TAG:-pk2}
mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
for KS in ${KERNELS:-k2_build:2 k2_scan:1 k_refine_level:2}; do
  K=${KS%%:*}; S=${KS##*:}
  $NCU --set full --clock-control none --import-source on -k regex:"$K" -c 1 --launch-skip $S \
    -o /tmp/$K -f python bench.py --config ${CFG:-C4} --res ${RES:-32} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $T/$K.log 2>&1
  $NCU -i /tmp/$K.ncu-rep --page raw --csv > $T/$K.raw.csv 2>/dev/null
  $NCU -i /tmp/$K.ncu-rep --page details > $T/$K.details.txt 2>/dev/null
  $NCU -i /tmp/$K.ncu-rep --page source --csv --print-source sass > $T/$K.sass.csv 2>/dev/null
  $NCU -i /tmp/$K.ncu-rep --page source --csv > $T/$K.src.csv 2>/dev/null
done
ls -la $T
