set -x
O=gpurun_out/s3u
mkdir -p $O
timeout 600 python scripts/sssp_prof.py 2883584 134217728 1073741824 > $O/new_lb4.txt 2>&1; cat $O/new_lb4.txt | tail -3
