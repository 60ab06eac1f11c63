# ncu --set full of one SSSP pull-round launch (rmat:24)
set -x
O=gpurun_out/s3s
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_sssp_pull_tiles' -s 10 -c 1 -o $O/sssp_pull python scripts/sssp_prof.py 134217728 > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu.log
