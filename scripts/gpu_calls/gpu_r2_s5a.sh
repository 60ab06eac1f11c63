# ncu --set full of the CC union pass (k_cc_edges) at rmat:24
set -x
O=gpurun_out/s5a
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cc_edges -c 1 -o $O/cc python scripts/traversal_spans.py 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
