set -u
D=gpurun_out/s2/k1g; mkdir -p $D
PROBE="python tools/gpu_probe.py c2 --reps 2 --device-gen --geo on"
$PROBE > $D/probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused2_kernel -s 1 -c 1 -f -o $D/k1g_c2 $PROBE > $D/full.log 2>&1; echo "full rc=$?"
