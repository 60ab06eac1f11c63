# SSSP pull: dist loads through L1 (__ldg, GCB_SSSP_DIST_L1=1) vs L2-only (__ldcg, shipped); parity and device spans
O=gpurun_out/s6j
mkdir -p $O
GCB_SSSP_DIST_L1=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -q -p no:cacheprovider -k "sssp or SSSP" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for i in 1 2; do
timeout 600 python scripts/traversal_spans.py 7 > $O/base$i.txt 2>&1; echo "ldcg: $(tail -1 $O/base$i.txt)"
GCB_SSSP_DIST_L1=1 timeout 600 python scripts/traversal_spans.py 7 > $O/l1$i.txt 2>&1; echo "ldg: $(tail -1 $O/l1$i.txt)"
done
