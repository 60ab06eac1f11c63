# round-2 sanitizer follow-up (final kernel set): racecheck of the
# shared-memory kernels (hot tables, the packed hub kernel's fixed-point table
# and per-warp row slices, the live-range update) with the host loop;
# synccheck of the suites without the graph-loop test (a CUDA-graph WHILE
# body; run on its own below, after the k_merge barrier fix); memcheck of the
# new paths.
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/r2_sanitizer_d
mkdir -p $O
F="tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_gcb.py"
GCB_NO_GRAPH=1 timeout 1500 $CS --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "FastLayouts or Overlapped or push" > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
for t in synccheck racecheck memcheck; do
  timeout 600 $CS --tool $t --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k graph_loop > $O/graph_loop_$t.log 2>&1; echo "rc=$?" >> $O/graph_loop_$t.log
done
GCB_NO_GRAPH=1 timeout 1200 $CS --tool synccheck --error-exitcode 99 python -m pytest $F -m gpu -q -p no:cacheprovider -k "not graph_loop" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "FastLayouts or Sharded" > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
