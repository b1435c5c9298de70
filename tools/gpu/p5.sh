# ncu --set full: K1g on C3 and C5 (3 CTAs/SM), K1s on C4 (node program 1)
O=gpurun_out/p5; mkdir -p $O
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
for cfg in c3 c5; do
  P="python tools/kbench.py $cfg --reps 2"
  $P > $O/plain_$cfg.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused2 -s 3 -c 1 --metrics $M -f -o $O/k1g_$cfg $P > $O/ncu_$cfg.log 2>&1
  echo "$cfg ncu rc=$?"
done
P="python tools/kbench.py c4 --reps 2"
$P > $O/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -f -o $O/k1s_c4 $P > $O/ncu_c4.log 2>&1
echo "c4 ncu rc=$?"
P="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$P > $O/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $P > $O/ncu_launches.log 2>&1
echo "launches rc=$?"
