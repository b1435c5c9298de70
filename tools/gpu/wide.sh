O=gpurun_out/wide; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2; do
  NKB_K1G_WIDE=0 python tools/kbench.py c2 --reps 40 --tag w256 >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 --reps 40 --tag w384 >> $O/kb.jsonl 2>> $O/kb.err
  NKB_K1G_OCC=2 python tools/kbench.py c3 c5 --reps 30 --tag occ2_w384 >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c3 c5 --reps 30 --tag occ3_w256 >> $O/kb.jsonl 2>> $O/kb.err
done
cat $O/kb.jsonl; tail -2 $O/pytest.log
