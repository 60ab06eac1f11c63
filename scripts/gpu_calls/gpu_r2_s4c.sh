# pull-gather ablations (instrumented build): cost of the per-row reduction and the stores
set -x
O=gpurun_out/s4c
mkdir -p $O
L=$PWD/paper_1904_02241_b200/libgcb_b200_abl.so
GCB_LIB=$L timeout 900 python scripts/variants.py 24 "full:GCB_ABL=0;warpsum:GCB_ABL=4;nostore:GCB_ABL=1;nogather:GCB_ABL=2;skeleton:GCB_ABL=7" 20 2 > $O/abl.txt 2>&1; cat $O/abl.txt | tail -11
