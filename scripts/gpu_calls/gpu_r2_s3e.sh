# bank-sorted hub tiles: parity, A/B, graph-loop synccheck after the k_merge init fix, ncu
set -x
O=gpurun_out/s3e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or headline or rmat24 or MidScale" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 900 python scripts/variants.py 24 "sorted:_FRESH=1;arena:_FRESH=1,GCB_HUB_NOSORT=1" 20 3 > $O/variants.txt 2>&1; tail -7 $O/variants.txt
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k graph_loop > $O/graph_loop_synccheck.log 2>&1; echo "rc=$?" >> $O/graph_loop_synccheck.log; tail -4 $O/graph_loop_synccheck.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_push_hub' -s 10 -c 1 -o $O/hub python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu.log
