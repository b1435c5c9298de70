set -u
D=gpurun_out/s2; mkdir -p $D
for L in prev cur; do
  if [ $L = prev ]; then export NKB_LIB=$PWD/paper_2312_09888_b200/lib/libnekb200_prev.so; else unset NKB_LIB; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pairwise_chunk -s 1 -c 1 -f -o $D/stats_$L python tools/stats_probe.py c4 --reps 1 > $D/stats_ncu_$L.log 2>&1; echo "$L rc=$?"
done
