set -u
mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s2/pytest_gpu2.log
for v in 1 0; do
  NKB_STREAM=$v timeout 300 python tools/gpu_probe.py c4 --reps 4 --device-gen --geo off > gpurun_out/s2/c4_stream$v.log 2>&1; echo "c4 stream=$v rc=$?"
  grep "rep 3" gpurun_out/s2/c4_stream$v.log
done
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2/c4_bench.json 2> gpurun_out/s2/c4_bench.err; echo "bench c4 rc=$?"
