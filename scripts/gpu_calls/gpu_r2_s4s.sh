# P=8 degree-ordered shards: hybrid everywhere (GCB_HYBRID=2) and 24576 hubs vs the cost model
set -x
O=gpurun_out/s4s
mkdir -p $O
run() {
  env DO=1 CALIB=1 "$@" timeout 600 python scripts/shard_estimate.py 24 8 > $O/shards_$1.json 2>&1
  python -c "
import json,sys
d=json.loads(open('$O/shards_$1.json').read().strip().splitlines()[-1])
for k in ('model_cuts','calibrated_cuts'):
  x=d[k]; print('$1',k,'max',max(x['step_ms_per_shard']),'sum',x['sum_of_steps_ms'],x['estimate_ms_per_iteration_at_900GBps'],x['step_ms_per_shard'],[p['hub_push'] for p in x['kernel_ms_per_shard_step']])
"
}
run GCB_HYBRID=1
run GCB_HYBRID=2
run GCB_HYBRID_HUBS=24576
run GCB_HYBRID=2 GCB_HYBRID_HUBS=24576
