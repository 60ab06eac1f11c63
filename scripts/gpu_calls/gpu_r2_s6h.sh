# SSSP pull with the frontier's distances in fdist (GCB_SSSP_FDIST=1) vs bitmap + dist: parity and device spans
O=gpurun_out/s6h
mkdir -p $O
GCB_SSSP_FDIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -q -p no:cacheprovider -k "sssp or SSSP" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
for i in 1 2; do
timeout 600 python scripts/traversal_spans.py 7 > $O/base$i.txt 2>&1; echo "base: $(tail -1 $O/base$i.txt)"
GCB_SSSP_FDIST=1 timeout 600 python scripts/traversal_spans.py 7 > $O/fd$i.txt 2>&1; echo "fdist: $(tail -1 $O/fd$i.txt)"
done
GCB_SSSP_FDIST=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_fd.csv python scripts/sssp_once.py > $O/ncu1.log 2>&1; echo "ncu rc=$?"
