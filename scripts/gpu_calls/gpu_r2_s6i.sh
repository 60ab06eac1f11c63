# SSSP pull occupancy A/B: __launch_bounds__(256, MINB) for MINB 4 (shipped) / 5 / 6 / 8, device spans at rmat:24
O=gpurun_out/s6i
mkdir -p $O
for i in 1 2; do for M in 4 5 6 8; do
GCB_SSSP_MINB=$M timeout 600 python scripts/traversal_spans.py 7 > $O/m$M.$i.txt 2>&1; echo "minb $M: $(tail -1 $O/m$M.$i.txt)"
done; done
GCB_SSSP_MINB=6 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "sssp or SSSP" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
