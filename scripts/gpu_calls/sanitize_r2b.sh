# round-2 sanitizer follow-up: finish the synccheck sweep without the
# CUDA-graph test, isolate the graph-loop synccheck reports, racecheck the
# suites the first sweep did not reach (acceptance, GCB container, new tests)
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/r2_sanitizer_b
mkdir -p $O
F="tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_gcb.py"
GCB_NO_GRAPH=1 timeout 1500 $CS --tool synccheck python -m pytest $F -m gpu -q -p no:cacheprovider -k "not graph_loop" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
for m in host graph; do timeout 300 $CS --tool synccheck python scripts/sync_graph_loop.py $m > $O/synccheck_loop_$m.log 2>&1; echo "rc=$?" >> $O/synccheck_loop_$m.log; done
GCB_NO_GRAPH=1 timeout 2400 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_gcb.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "acceptance or gcb or Overlapped or degree_ordered or pack_unpack or c2 or c6" > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
for f in $O/*.log; do echo "== $f"; tail -5 $f; done
