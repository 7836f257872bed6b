export SPOLY_PARITY_LOG=gpurun_out/parity4.jsonl
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/gputest4.log 2>&1; echo PYTEST_EXIT $?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo BENCH $?
for c in C3 C4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench4_$c.json 2>> gpurun_out/bench4.err; done
SPOLY_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4_mp.json 2> gpurun_out/bench4_mp.err; echo MP $?
