# live-range update + isolated-tail permute: parity, A/B, bench, ncu source capture
set -x
O=gpurun_out/s3b
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
timeout 600 python scripts/variants.py 24 "live:;full:GCB_FULL_UPDATE=1" 20 3 > $O/variants.txt 2>&1; tail -8 $O/variants.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.log 2> $O/bench.err; echo "bench rc=$?"
tail -c 3000 $O/bench.log; tail -3 $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_pull_hot|k_push_hub|k_pr_update2|k_permute_out|k_pr_init' -s 40 -c 6 -o $O/full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $O/ncu.log
