# edge-parallel relabel + in-degrees counted per local row: promotion trace, layout parity tests
O=gpurun_out/s6e
mkdir -p $O
timeout 600 python scripts/promotion_trace.py 24 > $O/promo.txt 2>&1; echo "promo rc=$?"; tail -30 $O/promo.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -q -p no:cacheprovider -k "FastLayouts or promotion or default_pipeline or hybrid or Sharded or rmat24_pr or push" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
