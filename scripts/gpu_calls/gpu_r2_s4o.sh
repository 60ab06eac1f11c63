set -x
O=gpurun_out/s4o
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or Spmv or c2" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 900 python scripts/variants.py 24 "full_tiles:" 20 3 > $O/ab.txt 2>&1; tail -3 $O/ab.txt
