# per-call work trimmed to the connected range: parity + timing
set -x
O=gpurun_out/s3q
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or rmat24_pagerank or MidScale or PageRank" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 600 python scripts/variants.py 24 "trim:;full:GCB_FULL_UPDATE=1" 20 3 > $O/variants.txt 2>&1; tail -6 $O/variants.txt
