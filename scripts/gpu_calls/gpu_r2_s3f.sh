# per-shard steps at P = 8 (rmat:24) after the hub-kernel work, both shard layouts; racecheck of the bank sort
set -x
O=gpurun_out/s3f
mkdir -p $O
timeout 600 python scripts/shard_estimate.py 24 8 > $O/shards.json 2>&1; tail -c 600 $O/shards.json
DO=1 timeout 600 python scripts/shard_estimate.py 24 8 > $O/shards_do.json 2>&1; tail -c 600 $O/shards_do.json
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "Sharded or peer" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
GCB_NO_GRAPH=1 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "hybrid_split or live_range" > $O/racecheck_hub.log 2>&1; echo "rc=$?" >> $O/racecheck_hub.log; tail -3 $O/racecheck_hub.log
