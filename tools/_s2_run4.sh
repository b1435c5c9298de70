set -u
D=gpurun_out/s2; mkdir -p $D
for c in c2 c4; do
  for L in prev cur; do
    if [ $L = prev ]; then export NKB_LIB=$PWD/paper_2312_09888_b200/lib/libnekb200_prev.so; else unset NKB_LIB; fi
    timeout 300 python tools/stats_probe.py $c --reps 10 > $D/stats_${c}_$L.log 2>&1; echo "$c $L rc=$?"; cat $D/stats_${c}_$L.log | grep MB
  done
done
unset NKB_LIB
timeout 900 python -m pytest tests/test_gpu_stats.py -q -x > $D/pytest_stats.log 2>&1; echo "pytest stats rc=$?"; tail -2 $D/pytest_stats.log
