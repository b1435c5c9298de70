# ncu capture of the compact-geometry K1g (C2) + FP64 instruction counts; GPU suite first
O=gpurun_out/p1; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
PROBE="python tools/gpu_probe.py c2 --reps 2 --device-gen --geo on"
$PROBE > $O/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused2 -s 1 -c 1 \
    --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -f -o $O/fused2_c2 $PROBE > $O/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 $O/pytest.log
