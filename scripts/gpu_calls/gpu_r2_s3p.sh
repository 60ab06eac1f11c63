# dynamic (chunked) tile order in the hub pass: parity, timing, ncu active cycles
set -x
O=gpurun_out/s3p
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or Sharded or rmat24_pagerank or MidScale or live" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 600 python scripts/variants.py 24 "base:" 20 3 > $O/variants.txt 2>&1; tail -3 $O/variants.txt
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,sm__cycles_active.min,sm__cycles_active.max --clock-control none -k regex:'k_push_hub|k_pull_hot' -s 20 -c 4 --csv --log-file $O/active.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu.log 2>&1; echo "ncu rc=$?"
