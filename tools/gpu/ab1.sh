# A/B: prev (HEAD~) vs new library on the kernel-level step; GPU suite on new
O=gpurun_out/ab1; mkdir -p $O
L=paper_2312_09888_b200/lib
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2; do
  NKB_LIB=$L/libnekb200_prev.so python tools/kbench.py c2 c3 c4 --reps 30 --tag prev >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 c3 c4 --reps 30 --tag new >> $O/kb.jsonl 2>> $O/kb.err
  NKB_STREAM_L2AHEAD=0 python tools/kbench.py c4 --reps 30 --tag new_noahead >> $O/kb.jsonl 2>> $O/kb.err
done
python tools/kbench.py c5 --elements 65536 --reps 20 --tag new >> $O/kb.jsonl 2>> $O/kb.err
tail -2 $O/pytest.log; cat $O/kb.jsonl
