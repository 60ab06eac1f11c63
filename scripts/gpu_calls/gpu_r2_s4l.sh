set -x
O=gpurun_out/s4l
mkdir -p $O
GCB_RELABEL_AFTER=20 timeout 600 python scripts/promotion_cost.py > $O/promo.txt 2>&1; cat $O/promo.txt
GCB_RELABEL_AFTER=20 timeout 600 python scripts/promotion_cost.py > $O/promo2.txt 2>&1; cat $O/promo2.txt
