set -u
D=gpurun_out/s2/r10; mkdir -p $D
for c in c1 c2 c4; do
  G=""; [ $c != c1 ] && G="--device-gen"
  NKB_LIB=$PWD/paper_2312_09888_b200/lib/libnekb200_prev.so timeout 600 python tools/gpu_probe.py $c --reps 4 $G --geo on > $D/${c}_prev.log 2>&1
  echo "$c prev: $(grep 'rep 3' $D/${c}_prev.log | grep -o 'raster [0-9.]*')"
  for B in 16 64 256 100000000; do
    NKB_RASTER_BIG_BOX=$B timeout 600 python tools/gpu_probe.py $c --reps 4 $G --geo on > $D/${c}_$B.log 2>&1
    echo "$c big=$B: $(grep 'rep 3' $D/${c}_$B.log | grep -o 'raster [0-9.]*')"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s2/r10/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/s2/r10/pytest_parity.log
