# degree-ordered shards with the hybrid hub pass forced (the cost model predates the packed hub kernel)
set -x
O=gpurun_out/s3g
mkdir -p $O
DO=1 GCB_HYBRID=2 timeout 600 python scripts/shard_estimate.py 24 8 > $O/shards_do_hyb.json 2>&1; tail -c 300 $O/shards_do_hyb.json
for S in 21 22; do
timeout 600 python scripts/variants.py $S "auto:_FRESH=1;hyb:_FRESH=1,GCB_HYBRID=2;nohyb:_FRESH=1,GCB_HYBRID=0" 20 2 > $O/variants_$S.txt 2>&1; tail -6 $O/variants_$S.txt
done
