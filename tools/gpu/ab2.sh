# node programs on/off (same library) + GPU suite
O=gpurun_out/ab2; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2; do
  NKB_NODE_PROGS=0 python tools/kbench.py c2 c3 --reps 30 --tag generic >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 c3 --reps 30 --tag progs >> $O/kb.jsonl 2>> $O/kb.err
done
python tools/kbench.py c5 --elements 65536 --reps 20 --tag progs >> $O/kb.jsonl 2>> $O/kb.err
tail -2 $O/pytest.log; cat $O/kb.jsonl
