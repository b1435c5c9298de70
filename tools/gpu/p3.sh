O=gpurun_out/p3; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2 3; do python tools/kbench.py c2 c3 c5 --reps 40 --tag new >> $O/kb.jsonl 2>> $O/kb.err; done
cat $O/kb.jsonl
PROBE="python tools/gpu_probe.py c2 --reps 2 --device-gen --geo on"
$PROBE > $O/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused2 -s 1 -c 1 \
    --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -f -o $O/fused2_c2 $PROBE > $O/ncu.log 2>&1
echo "ncu rc=$?"; tail -2 $O/pytest.log
