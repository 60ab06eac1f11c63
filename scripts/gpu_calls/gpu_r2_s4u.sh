# A/B: double-buffered pull (k_pull_db: next tile's gathers issued before the reduction) at 16/20/24/28 warps vs k_pull_hot
set -x
O=gpurun_out/s4u
mkdir -p $O
GCB_PULL_DB=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or live_range or hybrid" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
P=paper_1904_02241_b200
for r in 1 2; do
  timeout 600 python scripts/variants.py 24 "base:;db24:GCB_PULL_DB=1;base_hb:GCB_NO_RELABEL=1;db24_hb:GCB_PULL_DB=1,GCB_NO_RELABEL=1" 20 1 >> $O/ab.txt 2>&1
  for w in 16 20 28; do
    GCB_LIB=$P/libgcb_b200_db$w.so timeout 600 python scripts/variants.py 24 "db$w:GCB_PULL_DB=1;db${w}_hb:GCB_PULL_DB=1,GCB_NO_RELABEL=1" 20 1 >> $O/ab.txt 2>&1
  done
done
grep -E "^r" $O/ab.txt
