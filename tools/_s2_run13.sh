set -u
D=gpurun_out/s2/r13; mkdir -p $D
for c in c2 c3; do
  for L in prev cur cur8; do
    unset NKB_LIB NKB_STAGE16
    [ $L = prev ] && export NKB_LIB=$PWD/paper_2312_09888_b200/lib/libnekb200_prev.so
    [ $L = cur8 ] && export NKB_STAGE16=0
    timeout 600 python tools/gpu_probe.py $c --reps 5 --device-gen --geo on > $D/${c}_$L.log 2>&1
    echo "$c $L: $(grep 'rep [234]' $D/${c}_$L.log | grep -o 'fused [0-9.]*' | tr '\n' ' ')"
  done
done
unset NKB_LIB NKB_STAGE16
for L in prev cur; do
  [ $L = prev ] && export NKB_LIB=$PWD/paper_2312_09888_b200/lib/libnekb200_prev.so
  NKB_STREAM=0 timeout 600 python tools/gpu_probe.py c4 --reps 3 --device-gen --geo off > $D/c4k1_$L.log 2>&1
  echo "c4 K1 $L: $(grep 'rep [12]' $D/c4k1_$L.log | grep -o 'fused [0-9.]*' | tr '\n' ' ')"
  unset NKB_LIB
done
timeout 1200 python -m pytest tests -m gpu -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $D/pytest.log
