# CC without the per-edge source array (edge groups, shuffle row search fused with the union pass): parity + device spans
set -x
O=gpurun_out/s4x
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "cc or CC or components or twitter" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 600 python scripts/traversal_spans.py 5 > $O/spans.txt 2>&1; tail -2 $O/spans.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cc --csv --log-file $O/cc_launches.csv python scripts/traversal_spans.py 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
