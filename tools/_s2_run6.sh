set -u
D=gpurun_out/s2; mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pairwise_chunk -s 1 -c 1 -f -o $D/stats_v3 python tools/stats_probe.py c4 --reps 1 > $D/stats_ncu_v3.log 2>&1; echo "rc=$?"
