O=gpurun_out/rlanes; rm -rf $O; mkdir -p $O
NKB_RASTER_LANES=4 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render.py -m gpu -q -x > $O/pytest4.log 2>&1; echo "pytest4 rc=$?" >> $O/pytest4.log; tail -n 2 $O/pytest4.log
NKB_RASTER_LANES=2 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "raster or c1 or box" > $O/pytest2.log 2>&1; echo "pytest2 rc=$?" >> $O/pytest2.log; tail -n 2 $O/pytest2.log
for r in 1 2; do
  for L in 1 2 4; do NKB_RASTER_LANES=$L python tools/kbench.py c1 c2 c3 c5 --reps 20 --tag L$L >> $O/kb.jsonl 2>> $O/kb.err; done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open('gpurun_out/rlanes/kb.jsonl'):
    j = json.loads(l); d[(j['config'], j['tag'])].append(j['raster'])
for k in sorted(d): print(k, d[k])
PY
