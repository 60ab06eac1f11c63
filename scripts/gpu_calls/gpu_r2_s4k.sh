# hub fixed-point scale 2^-62 (default) vs 2^-58 / 2^-56 (zero high-word adds skipped): time and error
set -x
O=gpurun_out/s4k
mkdir -p $O
timeout 600 python scripts/variants.py 24 "fix62:" 20 2 > $O/fix62.txt 2>&1; tail -2 $O/fix62.txt
for S in 58 56; do
  GCB_LIB=$PWD/paper_1904_02241_b200/libgcb_b200_fix$S.so timeout 600 python scripts/variants.py 24 "fix$S:" 20 2 > $O/fix$S.txt 2>&1; tail -2 $O/fix$S.txt
done
