# configs[4] on one GPU with the round-2 kernels: PageRank bench line and CC at rmat:25:44:1
set -x
O=gpurun_out/s3o
mkdir -p $O
timeout 1200 python bench.py --scale 25 --edge-factor 44 --steps 10 --warmup 3 --no-secondary > $O/bench_tw.log 2> $O/bench_tw.err; echo "bench rc=$?"; tail -c 2500 $O/bench_tw.log; tail -3 $O/bench_tw.err
timeout 900 python scripts/twitter_scale.py > $O/cc_tw.log 2>&1; echo "cc rc=$?"; tail -5 $O/cc_tw.log
