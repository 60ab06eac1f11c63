# 64-row destination-id cache in the pull gather: parity and A/B
set -x
O=gpurun_out/s3k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or Spmv or MidScale" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 900 python scripts/variants.py 24 "ids64:_FRESH=1;ids32:_FRESH=1,GCB_PULL_IDS=32" 20 3 > $O/variants24.txt 2>&1; tail -6 $O/variants24.txt
timeout 900 python scripts/variants.py 22 "ids64:_FRESH=1;ids32:_FRESH=1,GCB_PULL_IDS=32" 20 3 > $O/variants22.txt 2>&1; tail -6 $O/variants22.txt
