# hub-count marginal rule (GCB_HYBRID_MIN_DEG): P=8 degree-ordered shard steps and the unsharded headline
set -x
O=gpurun_out/s4r
mkdir -p $O
for T in 0 600 1500 3000; do
  DO=1 CALIB=1 GCB_HYBRID_MIN_DEG=$T timeout 600 python scripts/shard_estimate.py 24 8 > $O/shards_T$T.json 2>&1
  python -c "
import json,sys
d=json.loads(open('$O/shards_T$T.json').read().strip().splitlines()[-1])
for k in ('model_cuts','calibrated_cuts'):
  x=d[k]; print('T=$T',k,'max',max(x['step_ms_per_shard']),'sum',x['sum_of_steps_ms'],x['estimate_ms_per_iteration_at_900GBps'],[p['hub_push'] for p in x['kernel_ms_per_shard_step']])
"
done
timeout 900 python scripts/variants.py 24 "T0:_FRESH=1,GCB_HYBRID_MIN_DEG=0;T1500:_FRESH=1,GCB_HYBRID_MIN_DEG=1500;T3000:_FRESH=1,GCB_HYBRID_MIN_DEG=3000" 20 2 > $O/ab.txt 2>&1; tail -7 $O/ab.txt
