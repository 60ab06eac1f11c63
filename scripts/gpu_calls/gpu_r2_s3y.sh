# window missProp normal vs streaming: timing and DRAM bytes of the pull launch (ncu, warm L2: --cache-control none)
set -x
O=gpurun_out/s3y
mkdir -p $O
timeout 300 python scripts/variants.py 24 "normal:;stream:GCB_L2_WINDOW_STREAM=1" 20 3 > $O/variants.txt 2>&1; tail -6 $O/variants.txt
for V in normal stream; do
  if [ $V = stream ]; then export GCB_L2_WINDOW_STREAM=1; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'k_pull_hot' -s 30 -c 3 --csv --log-file $O/traffic_$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_$V.log 2>&1
  timeout 600 ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'k_pull_hot' -s 30 -c 3 --csv --log-file $O/traffic_warm_$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_warm_$V.log 2>&1
done
