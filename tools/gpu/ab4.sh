O=gpurun_out/ab4; mkdir -p $O
for r in 1 2; do
  NKB_EMIT_PREFETCH=0 python tools/kbench.py c2 c3 c5 --reps 30 --tag nopf >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 c3 c5 --reps 30 --tag pf >> $O/kb.jsonl 2>> $O/kb.err
done
cat $O/kb.jsonl
PROBE="python tools/kbench.py c5 --reps 2"
$PROBE > $O/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused2 -s 3 -c 1 \
    --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -f -o $O/fused2_c5 $PROBE > $O/ncu.log 2>&1
echo "ncu rc=$?"
