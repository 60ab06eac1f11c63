# round-2 session-3 check after the container rebuild: GPU suite, the opt-in
# Twitter-scale parity, the bench line, the ncu launch list of the bench
set -x
O=gpurun_out/s3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q --capture=sys --durations=30 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -40 $O/pytest.log
GCB_FULL_SCALE=1 timeout 900 python -m pytest tests/test_gpu_full_scale.py -m gpu -v --durations=0 -p no:cacheprovider > $O/full_scale.log 2>&1; echo "rc=$?" >> $O/full_scale.log
tail -12 $O/full_scale.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.log 2> $O/bench.err; echo "bench rc=$?"
tail -c 5000 $O/bench.log; tail -5 $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_launch.log 2>&1; echo "ncu rc=$?"
