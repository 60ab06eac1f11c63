# intermediate updates clear only the sums the next pass adds onto: parity and A/B
set -x
O=gpurun_out/s4g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or MidScale or rmat24_pagerank or access_policy" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 900 python scripts/variants.py 24 "zb:;full:GCB_FULL_CLEAR=1" 20 3 > $O/ab.txt 2>&1; tail -6 $O/ab.txt
