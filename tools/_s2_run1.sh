set -u
mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s2/pytest_gpu.log
for c in c2 c3 c4; do
  NKB_PROFILE_PHASES=1 timeout 300 python tools/gpu_probe.py $c --reps 3 --device-gen --geo on > gpurun_out/s2/phases_$c.log 2>&1; echo "$c rc=$?"
done
