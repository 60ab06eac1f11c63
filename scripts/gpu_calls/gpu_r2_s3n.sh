# multi-rank bench path (2 ranks on one GPU over gloo: a function check, not a speed number)
# with degree-ordered shards, dead-skip steps and the calibrated re-cut; P2P and NCCL-style exchange
set -x
O=gpurun_out/s3n
mkdir -p $O
GCB_DEVICE=0 GCB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 20 --steps 5 --warmup 3 > $O/bench2.log 2>&1; echo "bench2 rc=$?"; tail -c 1500 $O/bench2.log
GCB_EXCHANGE=nccl GCB_DEVICE=0 GCB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --scale 20 --steps 5 --warmup 3 > $O/bench2_sparse.log 2>&1; echo "bench2 sparse rc=$?"; tail -c 600 $O/bench2_sparse.log
timeout 900 python -m pytest tests/test_gpu_peer_exchange.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "peer or Sharded" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
