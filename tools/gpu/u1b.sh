O=gpurun_out/u1b; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
L=paper_2312_09888_b200/lib
for r in 1 2 3; do
  NKB_LIB=$L/libnekb200_prev.so python tools/kbench.py c1 c3 c5 --reps 20 --tag head >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c1 c3 c5 --reps 20 --tag u1 >> $O/kb.jsonl 2>> $O/kb.err
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open('gpurun_out/u1b/kb.jsonl'):
    j = json.loads(l); d[(j['config'], j['tag'])].append(j['fused'])
for k in sorted(d): print(k, d[k])
PY
