# L2 residency of the cold gathers: per-load range policy (default) vs a launch access-policy
# window over the head of the degree-ordered slice with a persisting set-aside of S MB
set -x
O=gpurun_out/s3v
mkdir -p $O
timeout 300 python scripts/variants.py 24 "range:" 20 2 > $O/range.txt 2>&1; tail -2 $O/range.txt
for S in 8 16 32 48; do
  GCB_L2_PERSIST=$S timeout 300 python scripts/variants.py 24 "win$S:" 20 2 > $O/win$S.txt 2>&1; tail -2 $O/win$S.txt
done
