# bulk L2 prefetch of the pull arena two tiles ahead: A/B and the ablation skeleton
set -x
O=gpurun_out/s4d
mkdir -p $O
timeout 900 python scripts/variants.py 24 "pf:;nopf:GCB_NO_L2_PREFETCH=1" 20 3 > $O/ab.txt 2>&1; tail -6 $O/ab.txt
L=$PWD/paper_1904_02241_b200/libgcb_b200_abl.so
GCB_LIB=$L timeout 900 python scripts/variants.py 24 "skeleton:GCB_ABL=7;skeleton_nopf:GCB_ABL=7,GCB_NO_L2_PREFETCH=1;nogather:GCB_ABL=2" 20 2 > $O/abl.txt 2>&1; tail -6 $O/abl.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "FastLayouts or PageRank or Spmv" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
