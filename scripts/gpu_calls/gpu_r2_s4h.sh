# how much the hybrid hub pass buys on the degree-ordered copy (packed hub kernel), and the hot-bit layout's split
set -x
O=gpurun_out/s4h
mkdir -p $O
timeout 900 python scripts/variants.py 24 "hyb:_FRESH=1;nohyb:_FRESH=1,GCB_HYBRID=0" 20 2 > $O/ab.txt 2>&1; tail -4 $O/ab.txt
timeout 900 python scripts/variants.py 24 "hotbit:_FRESH=1,GCB_NO_RELABEL=1" 20 2 > $O/hotbit.txt 2>&1; tail -2 $O/hotbit.txt
