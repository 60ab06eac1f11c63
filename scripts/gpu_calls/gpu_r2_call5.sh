# validate the overlapped upload / pack kernels / ordered shards, then measure:
# e2e phases, L2 range-policy variants, per-shard steps, full bench
set -x
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "Overlapped or pack_unpack or TestSharded or upload or TestFastLayouts or peer" > $O/c5_pytest.log 2>&1; echo "rc=$?" >> $O/c5_pytest.log
tail -5 $O/c5_pytest.log
timeout 600 python scripts/e2e_breakdown.py 24 10 > $O/c5_e2e.txt 2>&1; tail -6 $O/c5_e2e.txt
timeout 900 python scripts/variants.py 24 "base:;r1_32:GCB_L2_RANGE=32:1;r2_32:GCB_L2_RANGE=32:2;r1_16:GCB_L2_RANGE=16:1;r1_48:GCB_L2_RANGE=48:1;r2_64:GCB_L2_RANGE=64:2" 20 3 > $O/c5_variants.txt 2>&1; tail -20 $O/c5_variants.txt
timeout 600 python scripts/shard_estimate.py 24 8 > $O/c5_shards.json 2>&1; tail -c 2500 $O/c5_shards.json
DO=1 timeout 600 python scripts/shard_estimate.py 24 8 > $O/c5_shards_do.json 2>&1; tail -c 2500 $O/c5_shards_do.json
GCB_DEVICE=0 GCB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 20 --steps 5 --warmup 3 > $O/c5_bench2.log 2>&1; echo "bench2 rc=$?"; tail -c 2000 $O/c5_bench2.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/c5_bench.log 2> $O/c5_bench.err; echo "bench rc=$?"; tail -c 6000 $O/c5_bench.log; tail -5 $O/c5_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_pull_hot|k_push_hub' -s 30 -c 2 -o $O/c5_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/c5_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $O/c5_ncu.log
timeout 300 ./scripts/mb_atoms > $O/c5_mb_atoms.txt 2>&1; cat $O/c5_mb_atoms.txt
