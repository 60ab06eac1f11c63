# BFS pull rows skip vertices already found in an earlier block of the level
set -x
O=gpurun_out/s4b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "bfs or BFS or c6 or Traversal or bc or BC" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 600 python scripts/traversal_spans.py > $O/spans.txt 2>&1; tail -2 $O/spans.txt
