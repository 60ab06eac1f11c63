set -x
O=gpurun_out/s3w
mkdir -p $O
timeout 300 python scripts/variants.py 24 "range:" 20 3 > $O/range.txt 2>&1
for S in 48 64 80 0; do
  GCB_L2_PERSIST=$S timeout 300 python scripts/variants.py 24 "win$S:" 20 3 > $O/win$S.txt 2>&1
done
python - <<'PY'
import torch; p=torch.cuda.get_device_properties(0); print("persistingL2CacheMaxSize", getattr(p,'persisting_l2_cache_max_size', None), "L2", p.L2_cache_size)
PY
