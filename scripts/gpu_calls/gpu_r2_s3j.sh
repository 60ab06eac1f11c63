# why is a small shard's pull slow? ncu of shard 7's k_pull_hot (rmat:24, DO shards)
set -x
O=gpurun_out/s3j
mkdir -p $O
DO=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_pull_hot' -s 100 -c 1 -o $O/shard7_pull python scripts/shard_estimate.py 24 8 > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu.log
