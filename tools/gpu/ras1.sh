# warp-cooperative raster for large triangles: parity tests + A/B raster stage (prev = HEAD build)
O=gpurun_out/ras1; rm -rf $O; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
L=paper_2312_09888_b200/lib
for r in 1 2; do
  NKB_LIB=$L/libnekb200_prev.so python tools/kbench.py c1 c2 c5 c4 --reps 20 --tag prev >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c1 c2 c5 c4 --reps 20 --tag new >> $O/kb.jsonl 2>> $O/kb.err
done
cat $O/kb.jsonl
