O=gpurun_out/ab3; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2; do
  NKB_NODE_PROGS=0 python tools/kbench.py c4 --reps 20 --tag generic896 >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c4 --reps 20 --tag prog896 >> $O/kb.jsonl 2>> $O/kb.err
  NKB_STREAM_THREADS=1024 python tools/kbench.py c4 --reps 20 --tag prog1024 >> $O/kb.jsonl 2>> $O/kb.err
done
tail -2 $O/pytest.log; cat $O/kb.jsonl
