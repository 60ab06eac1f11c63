# paired hub atomics + coalesced u64 flush: parity, hub-count sweep, bench, ncu
set -x
O=gpurun_out/s3d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or Sharded or headline or rmat24 or graph_loop or MidScale" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
timeout 900 python scripts/variants.py 24 "h20k:_FRESH=1,GCB_HYBRID_HUBS=20480;h24k:_FRESH=1,GCB_HYBRID_HUBS=24576;h16k:_FRESH=1,GCB_HYBRID_HUBS=16384" 20 2 > $O/variants.txt 2>&1; tail -7 $O/variants.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e --no-secondary > $O/bench.log 2> $O/bench.err; echo "bench rc=$?"
tail -c 1200 $O/bench.log; tail -3 $O/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_push_hub|k_hub_fold' -s 20 -c 2 -o $O/hub python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu.log
