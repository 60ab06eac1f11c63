# SSSP at rmat:24: direction sequence per capacity and the launch list of one call
set -x
O=gpurun_out/s3r
mkdir -p $O
timeout 600 python scripts/sssp_prof.py 2883584 16777216 134217728 1073741824 100000000000 > $O/sssp.txt 2>&1; cat $O/sssp.txt | tail -6
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/sssp_launches.csv python scripts/sssp_prof.py 134217728 > $O/ncu.log 2>&1; echo "ncu rc=$?"
