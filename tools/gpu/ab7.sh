O=gpurun_out/ab7; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2; do
  NKB_K1G_PG=0 python tools/kbench.py c2 c3 c5 --reps 30 --tag nopg >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 c3 c5 --reps 30 --tag pg >> $O/kb.jsonl 2>> $O/kb.err
  NKB_K1G_OCC=2 python tools/kbench.py c2 c3 c5 --reps 30 --tag pg_occ2 >> $O/kb.jsonl 2>> $O/kb.err
done
tail -2 $O/pytest.log; cat $O/kb.jsonl
