set -x
O=gpurun_out/s4j
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "bfs or BFS or c6 or Traversal or bc or BC or sssp or SSSP or rmat24_bfs" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 600 python scripts/traversal_spans.py 7 > $O/spans.txt 2>&1; tail -1 $O/spans.txt
