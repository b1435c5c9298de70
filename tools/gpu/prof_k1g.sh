O=gpurun_out/pk1g; rm -rf $O; mkdir -p $O
PROBE="python tools/kbench.py c2 --reps 2"
$PROBE > $O/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused2 -s 2 -c 1 \
    --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -f -o $O/fused2_c2 $PROBE > $O/ncu.log 2>&1
echo "ncu rc=$?"
