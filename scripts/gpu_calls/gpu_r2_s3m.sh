# calibrated cuts for degree-ordered shards (dead-skip steps)
set -x
O=gpurun_out/s3m
mkdir -p $O
DO=1 CALIB=1 timeout 900 python scripts/shard_estimate.py 24 8 > $O/shards_do_calib.json 2>&1; tail -c 300 $O/shards_do_calib.json
