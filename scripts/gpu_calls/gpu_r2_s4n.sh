set -x
O=gpurun_out/s4n
mkdir -p $O
timeout 900 python scripts/variants.py 24 "lo0:;sub:GCB_NO_LO0=1" 20 3 > $O/ab.txt 2>&1; tail -6 $O/ab.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or Spmv" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
