# A/B: TMA bulk-copy staging (natural layout) vs cp.async into the swizzled ring; parity of the TMA variant
O=gpurun_out/tma; mkdir -p $O
NKB_K1G_TMA=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "prog or box_pipelines or taylor or c2_full" > $O/pytest_tma.log 2>&1; echo "pytest(tma) rc=$?" >> $O/pytest_tma.log
for r in 1 2; do
  python tools/kbench.py c2 c3 c5 --reps 40 --tag ldgsts >> $O/kb.jsonl 2>> $O/kb.err
  NKB_K1G_TMA=1 python tools/kbench.py c2 c3 c5 --reps 40 --tag tma >> $O/kb.jsonl 2>> $O/kb.err
done
cat $O/kb.jsonl; tail -2 $O/pytest_tma.log
P="python tools/kbench.py c2 --reps 2"
NKB_K1G_TMA=1 $P > $O/plain.log 2>&1 && NKB_K1G_TMA=1 ncu --set full --clock-control none --import-source on -k regex:fused2 -s 3 -c 1 -f -o $O/k1g_c2_tma $P > $O/ncu.log 2>&1
echo "ncu rc=$?"
