# pipelined SSSP pull round: parity and A/B against the round-1 kernel
set -x
O=gpurun_out/s3t
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "sssp or SSSP" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 600 python scripts/sssp_prof.py 2883584 134217728 1073741824 > $O/new.txt 2>&1; cat $O/new.txt | tail -3
GCB_SSSP_PULL=0 timeout 600 python scripts/sssp_prof.py 2883584 134217728 1073741824 > $O/old.txt 2>&1; cat $O/old.txt | tail -3
