# A/B: tile_row loaded one more iteration ahead in k_pull_hot (default) vs GCB_TROW_AHEAD=0
set -x
O=gpurun_out/s4t
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or Spmv or c2 or hybrid or live_range" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
L=paper_1904_02241_b200/libgcb_b200_trow0.so
for r in 1 2; do
  timeout 600 python scripts/variants.py 24 "ahead:;ahead_hotbit:GCB_NO_RELABEL=1" 20 2 >> $O/ab.txt 2>&1
  GCB_LIB=$L timeout 600 python scripts/variants.py 24 "trow0:;trow0_hotbit:GCB_NO_RELABEL=1" 20 2 >> $O/ab.txt 2>&1
done
grep -E "ahead|trow0" $O/ab.txt
