O=gpurun_out/pres; rm -rf $O; mkdir -p $O
python tools/kbench.py c2 --reps 2 > $O/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:resolve_kernel -s 2 -c 1 -f -o $O/resolve_c2 python tools/kbench.py c2 --reps 2 > $O/ncu.log 2>&1
echo "ncu rc=$?"
