# round-2 sanitizer follow-up: synccheck of the suites without the graph-loop
# test (a CUDA-graph WHILE body; run on its own below), the graph loop after
# the k_merge barrier fix, and racecheck of the shared-memory kernels (hot
# tables, the two-word fixed-point hub table with its per-warp row slices,
# the overlapped upload, the live-range update) with the host loop.
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/r2_sanitizer_d
mkdir -p $O
F="tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_gcb.py"
GCB_NO_GRAPH=1 timeout 1500 $CS --tool synccheck --error-exitcode 99 python -m pytest $F -m gpu -q -p no:cacheprovider -k "not graph_loop" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
for t in synccheck racecheck memcheck; do
  timeout 600 $CS --tool $t --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k graph_loop > $O/graph_loop_$t.log 2>&1; echo "rc=$?" >> $O/graph_loop_$t.log
done
GCB_NO_GRAPH=1 timeout 2700 $CS --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -q -p no:cacheprovider -k "FastLayouts or Overlapped or hybrid or live_range or push or c2_pagerank_routes" > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
