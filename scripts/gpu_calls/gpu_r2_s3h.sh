# session-3 evidence refresh: whole GPU suite, bench line, ncu launch list (traffic), ncu --set full of the iteration kernels
set -x
O=gpurun_out/s3h
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.log 2> $O/bench.err; echo "bench rc=$?"
tail -c 800 $O/bench.log; tail -3 $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'k_pull_hot|k_push_hub|k_hub_fold|k_pr_update2' -s 30 -c 8 --csv --log-file $O/traffic.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_pull_hot|k_push_hub|k_pr_update2' -s 30 -c 3 -o $O/full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
