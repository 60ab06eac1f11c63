# promotion-build stage costs at rmat:24 (scripts/promotion_trace.py) + sanitizer pass over the CC hooking kernel
O=gpurun_out/s6b
mkdir -p $O
timeout 600 python scripts/promotion_trace.py 24 > $O/promo.txt 2>&1; echo "promo rc=$?"; cat $O/promo.txt | tail -40
CS=/usr/local/cuda/bin/compute-sanitizer
K="cc_ or CC or Components"
GCB_NO_GRAPH=1 timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$K" > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
GCB_NO_GRAPH=1 timeout 900 $CS --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$K" > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
GCB_NO_GRAPH=1 timeout 900 $CS --tool synccheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$K" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
