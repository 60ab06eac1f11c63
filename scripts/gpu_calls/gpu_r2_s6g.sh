# SSSP at rmat:24: per-launch times of one call, and ncu --set full of one pull-round launch
O=gpurun_out/s6g
mkdir -p $O
timeout 600 python scripts/sssp_once.py > $O/plain.txt 2>&1; echo "plain rc=$?"; tail -2 $O/plain.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum --clock-control none --csv --log-file $O/launches.csv python scripts/sssp_once.py > $O/ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_sssp_pull -s 3 -c 1 -o $O/pull python scripts/sssp_once.py > $O/ncu2.log 2>&1; echo "ncu2 rc=$?"
