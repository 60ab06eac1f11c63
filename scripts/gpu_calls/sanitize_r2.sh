# round-2 compute-sanitizer sweep over the final kernel set (GPU box):
# memcheck / racecheck / synccheck over the small-graph GPU suites, the
# CUDA-graph convergence loop off for racecheck (see profiles/r1_sanitizer.txt),
# then the racecheck + graph-loop crash on its own.
F="tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_gcb.py"
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/r2_sanitizer
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version --format=csv,noheader > $O/gpu.txt
timeout 1500 $CS --tool memcheck --leak-check no python -m pytest $F -m gpu -q -x -p no:cacheprovider > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
GCB_NO_GRAPH=1 timeout 2400 $CS --tool racecheck --racecheck-report hazard python -m pytest $F -m gpu -q -x -p no:cacheprovider > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
GCB_NO_GRAPH=1 timeout 1500 $CS --tool synccheck python -m pytest $F -m gpu -q -x -p no:cacheprovider > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
timeout 600 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k graph_loop > $O/racecheck_graphloop.log 2>&1; echo "rc=$?" >> $O/racecheck_graphloop.log
for f in $O/*.log; do echo "== $f"; tail -4 $f; done
