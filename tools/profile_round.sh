#!/bin/bash
# Run on the GPU box (via gpurun): plain bench, then the ncu launch list of the
# same command, then one --set full capture of the surface pass (K1g fused2_kernel for C2).  Outputs in
# gpurun_out/; summarise locally with tools/summarize_profiles.py.
set -u
TAG=${1:-r01}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
echo "launch list rc=$?"
PROBE="python tools/gpu_probe.py c2 --reps 2 --device-gen --geo on"
$PROBE > gpurun_out/${TAG}_probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 \
    -f -o gpurun_out/${TAG}_fused $PROBE > gpurun_out/${TAG}_full.log 2>&1
echo "full capture rc=$?"
