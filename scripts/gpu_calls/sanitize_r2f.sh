# sanitizer pass over the block-0 direct-index pull (k_pull_hot LO0 instance, session 4)
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/r2_sanitizer_f
mkdir -p $O
K="FastLayouts or live_range or hybrid_split or virtual_shards or Spmv"
GCB_NO_GRAPH=1 timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$K" > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
GCB_NO_GRAPH=1 timeout 1500 $CS --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "FastLayouts or live_range" > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
GCB_NO_GRAPH=1 timeout 1500 $CS --tool synccheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$K" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
