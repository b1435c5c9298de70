set -u
D=gpurun_out/s2; mkdir -p $D
for L in prev cur; do
  if [ $L = prev ]; then export NKB_LIB=$PWD/paper_2312_09888_b200/lib/libnekb200_prev.so; else unset NKB_LIB; fi
  timeout 300 python tools/export_probe.py c2 > $D/export_$L.log 2>&1; echo "$L rc=$?"; grep GB/s $D/export_$L.log
done
unset NKB_LIB
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu7.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest_gpu7.log
