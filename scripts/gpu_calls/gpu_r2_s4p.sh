# A/B: deferred per-tile row stores in k_pull_hot (default build) vs GCB_PULL_DEFER=0
set -x
O=gpurun_out/s4p
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or Spmv or c2 or Hybrid or hybrid" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
L=paper_1904_02241_b200/libgcb_b200_nodefer.so
for r in 1 2; do
  timeout 600 python scripts/variants.py 24 "defer:" 20 2 >> $O/ab.txt 2>&1
  GCB_LIB=$L timeout 600 python scripts/variants.py 24 "nodefer:" 20 2 >> $O/ab.txt 2>&1
done
grep -E "defer" $O/ab.txt
