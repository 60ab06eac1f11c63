# sanitizer pass over the kernels changed after r2_sanitizer: pipelined SSSP pull (byte weights),
# one-launch BFS pull, unrolled level commit, the trimmed PageRank init/update/permute,
# dead-skip shard steps
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/r2_sanitizer_e
mkdir -p $O
K="sssp or SSSP or bfs or BFS or Traversal or c6 or FastLayouts or Sharded or live_range"
GCB_NO_GRAPH=1 timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 99 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -q -p no:cacheprovider -k "$K" > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
GCB_NO_GRAPH=1 timeout 2400 $CS --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "sssp or SSSP or bfs or BFS or live_range or hybrid_split" > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
GCB_NO_GRAPH=1 timeout 1500 $CS --tool synccheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -q -p no:cacheprovider -k "$K" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
