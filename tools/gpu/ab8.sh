# kDirect K1g (C2: scalar + slice coordinate loaded per node, not staged) A/B + GPU suite
O=gpurun_out/ab8; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  NKB_K1G_DIRECT=0 python tools/kbench.py c2 --reps 30 --tag staged >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 --reps 30 --tag direct2 >> $O/kb.jsonl 2>> $O/kb.err
  NKB_K1G_OCC=3 python tools/kbench.py c2 --reps 30 --tag direct3 >> $O/kb.jsonl 2>> $O/kb.err
done
tail -2 $O/pytest.log; cat $O/kb.jsonl
