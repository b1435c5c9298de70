set -u
D=gpurun_out/s2/r11; mkdir -p $D
for c in c1 c2 c4; do
  G=""; [ $c != c1 ] && G="--device-gen"
  for L in prev cur; do
    if [ $L = prev ]; then export NKB_LIB=$PWD/paper_2312_09888_b200/lib/libnekb200_prev.so; else unset NKB_LIB; fi
    timeout 600 python tools/gpu_probe.py $c --reps 4 $G --geo on > $D/${c}_$L.log 2>&1
    echo "$c $L: $(grep 'rep 3' $D/${c}_$L.log | grep -o 'raster [0-9.]*')  $(grep 'rep 3' $D/${c}_$L.log | grep -o 'total [0-9.]*')"
  done
done
unset NKB_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_render.py -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $D/pytest.log
