# dead-skip shard steps: parity (virtual shards, peer exchange), shard estimate
set -x
O=gpurun_out/s3l
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer_exchange.py -m gpu -x -q -p no:cacheprovider -k "Sharded or peer or FastLayouts or relabel or degree" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
DO=1 timeout 600 python scripts/shard_estimate.py 24 8 > $O/shards_do.json 2>&1; tail -c 400 $O/shards_do.json
timeout 600 python scripts/variants.py 24 "base:" 10 2 > $O/variants.txt 2>&1; tail -2 $O/variants.txt
