export SPOLY_PARITY_LOG=gpurun_out/parity8.jsonl
timeout 1200 python -m pytest tests -m gpu -q -rf --durations=5 > gpurun_out/gputest8.log 2>&1; echo PYTEST_EXIT $?
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench8_C4.json 2>/dev/null
TOOLS="memcheck" timeout 1500 bash scripts/sanitize.sh
