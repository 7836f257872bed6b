export SPOLY_PARITY_LOG=gpurun_out/parity5.jsonl
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/gputest5.log 2>&1; echo PYTEST_EXIT $?
bash scripts/ab.sh > gpurun_out/ab.log 2>&1
