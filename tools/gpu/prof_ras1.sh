O=gpurun_out/pras1; rm -rf $O; mkdir -p $O
python tools/kbench.py c1 --reps 2 > $O/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:raster_kernel -s 2 -c 1 -f -o $O/raster_c1 python tools/kbench.py c1 --reps 2 > $O/ncu.log 2>&1
echo "ncu rc=$?"
