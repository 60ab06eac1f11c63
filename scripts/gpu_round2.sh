# round-2 GPU check: the whole -m gpu suite (timings), then the bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --capture=sys --durations=30 ${PYTEST_ARGS:-} > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
tail -60 gpurun_out/r2_pytest.log
if [ -z "${NO_BENCH:-}" ]; then
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
tail -c 6000 gpurun_out/r2_bench.log; tail -20 gpurun_out/r2_bench.err
fi
