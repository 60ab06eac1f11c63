# BFS at rmat:24: launch list of one call (after warm-up)
set -x
O=gpurun_out/s4a
mkdir -p $O
cat > /tmp/bfs1.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import paper_1904_02241_b200 as gcb
g = gcb.generate_rmat(24, 16, 1)
bgt = gcb.partition_tocab(gcb.transpose(g), "pull", 1 << 21)
for _ in range(3):
    r = gcb.bfs(g, 0, g_blocked=bgt)
print(r.directions, [len(l) for l in r.levels])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bfs_launches.csv python /tmp/bfs1.py > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu.log
