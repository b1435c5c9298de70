O=gpurun_out/ez1; rm -rf $O; mkdir -p $O
NKB_EARLY_Z=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render.py tests/test_gpu_partitions.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
for r in 1 2; do
  python tools/kbench.py c1 c2 c5 c4 --reps 20 --tag atomic >> $O/kb.jsonl 2>> $O/kb.err
  NKB_EARLY_Z=1 python tools/kbench.py c1 c2 c5 c4 --reps 20 --tag earlyz >> $O/kb.jsonl 2>> $O/kb.err
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open('gpurun_out/ez1/kb.jsonl'):
    j = json.loads(l); d[(j['config'], j['tag'])].append(j['raster'])
for k in sorted(d): print(k, d[k])
PY
