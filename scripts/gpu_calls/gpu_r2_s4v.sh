# launch list of BFS / SSSP / CC at rmat:24 (scripts/traversal_spans.py, 1 rep)
set -x
O=gpurun_out/s4v
mkdir -p $O
timeout 600 python scripts/traversal_spans.py 3 > $O/spans.txt 2>&1; cat $O/spans.txt | tail -5
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python scripts/traversal_spans.py 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
