set -u
D=gpurun_out/s2/r15; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $D/pytest.log
for c in c2 c3; do
  for v in 0 1; do
    NKB_FUSED2=$v timeout 600 python tools/gpu_probe.py $c --reps 5 --device-gen --geo on > $D/${c}_$v.log 2>&1
    echo "$c fused2=$v rc=$?: $(grep 'rep [234]' $D/${c}_$v.log | grep -o 'fused [0-9.]*' | tr '\n' ' ')"
  done
done
