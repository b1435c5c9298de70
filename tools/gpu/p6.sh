O=gpurun_out/p6; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2; do python tools/kbench.py c2 c3 c5 --reps 40 --tag triact >> $O/kb.jsonl 2>> $O/kb.err; done
cat $O/kb.jsonl; tail -2 $O/pytest.log
