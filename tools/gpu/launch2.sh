O=gpurun_out/launch2; rm -rf $O; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/b.json 2> $O/b.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
echo "ncu rc=$?"
