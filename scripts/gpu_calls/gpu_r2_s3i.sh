# batched hot-table staging: unsharded pull time and per-shard steps (shard 7 = few edges, many rows)
set -x
O=gpurun_out/s3i
mkdir -p $O
timeout 600 python scripts/variants.py 24 "base:" 20 3 > $O/variants.txt 2>&1; tail -3 $O/variants.txt
DO=1 timeout 600 python scripts/shard_estimate.py 24 8 > $O/shards_do.json 2>&1; tail -c 300 $O/shards_do.json
timeout 600 ncu --set full --clock-control none -k regex:'k_pull_hot' -s 50 -c 8 -o $O/shard_pull python scripts/shard_estimate.py 22 8 > $O/ncu.log 2>&1; echo "ncu rc=$?"
