O=gpurun_out/ab6; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2; do
  NKB_K1G_DIRECT=0 python tools/kbench.py c2 --reps 40 --tag staged >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 --reps 40 --tag direct >> $O/kb.jsonl 2>> $O/kb.err
  NKB_K1G_OCC=2 NKB_K1G_DIRECT=0 python tools/kbench.py c2 --reps 40 --tag occ2 >> $O/kb.jsonl 2>> $O/kb.err
done
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -2 $O/pytest.log; cat $O/kb.jsonl; python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['parity'])"
