# round-2 compute-sanitizer sweep over the final kernel set (GPU box):
# memcheck over the small-graph GPU suites; racecheck and synccheck with the
# CUDA-graph convergence loop off (GCB_NO_GRAPH=1: racecheck cannot follow a
# WHILE conditional node, see profiles/r1_sanitizer.txt); then the graph loop
# alone under memcheck/synccheck (scripts/sync_graph_loop.py host|graph).
F="tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_gcb.py"
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/r2_sanitizer
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version --format=csv,noheader > $O/gpu.txt
$CS --version | tail -1 >> $O/gpu.txt
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 99 python -m pytest $F -m gpu -q -p no:cacheprovider > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
GCB_NO_GRAPH=1 timeout 1800 $CS --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest $F -m gpu -q -p no:cacheprovider > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
GCB_NO_GRAPH=1 timeout 1200 $CS --tool synccheck --error-exitcode 99 python -m pytest $F -m gpu -q -p no:cacheprovider > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
for m in host graph; do
  for t in memcheck synccheck racecheck; do
    timeout 300 $CS --tool $t --error-exitcode 99 python scripts/sync_graph_loop.py $m > $O/loop_${m}_$t.log 2>&1; echo "rc=$?" >> $O/loop_${m}_$t.log
  done
done
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
