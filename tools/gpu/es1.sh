# emission coordinates staged into dead S_dv space (NKB_EMIT_STAGE) A/B + parity
O=gpurun_out/es1; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
for r in 1 2; do
  NKB_EMIT_STAGE=0 python tools/kbench.py c1 c2 c3 c5 --reps 20 --tag l2pf >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c1 c2 c3 c5 --reps 20 --tag stage >> $O/kb.jsonl 2>> $O/kb.err
done
cat $O/kb.jsonl
