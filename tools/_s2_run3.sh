set -u
D=gpurun_out/s2
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu3.log 2>&1; echo "pytest rc=$?"
tail -3 $D/pytest_gpu3.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 > $D/c4_bench3.json 2> $D/c4_bench3.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $D/c2_bench3.json 2> $D/c2_bench3.err; echo "bench c2 rc=$?"
CMD="python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-max-gb 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/c4_launches.csv $CMD > $D/c4_launches.log 2>&1; echo "launch list rc=$?"
PROBE="python tools/gpu_probe.py c4 --reps 2 --device-gen --geo off"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 -f -o $D/c4_stream $PROBE > $D/c4_full.log 2>&1; echo "full capture rc=$?"
