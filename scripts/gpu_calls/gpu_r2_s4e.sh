# 512-edge tiles in the promoted pull (k_pull_hot16): parity and A/B against 256-edge tiles
set -x
O=gpurun_out/s4e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or MidScale or rmat24_pagerank" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
timeout 900 python scripts/variants.py 24 "v16:;v8:GCB_PULL_V8=1" 20 3 > $O/ab24.txt 2>&1; tail -6 $O/ab24.txt
timeout 900 python scripts/variants.py 22 "v16:;v8:GCB_PULL_V8=1" 20 2 > $O/ab22.txt 2>&1; tail -4 $O/ab22.txt
