O=gpurun_out/res1; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_render.py tests/test_gpu_partitions.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
L=paper_2312_09888_b200/lib
for r in 1 2; do
  NKB_LIB=$L/libnekb200_prev.so python tools/kbench.py c1 c2 c5 --reps 20 --tag head >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c1 c2 c5 --reps 20 --tag px4 >> $O/kb.jsonl 2>> $O/kb.err
done
for r in 1 2; do
  NKB_LIB=$L/libnekb200_prev.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/head_$r.json 2>/dev/null
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/new_$r.json 2>/dev/null
done
python - <<'PY'
import json, collections, glob
d = collections.defaultdict(list)
for l in open('gpurun_out/res1/kb.jsonl'):
    j = json.loads(l); d[(j['config'], j['tag'])].append(j['resolve'])
for k in sorted(d): print(k, d[k])
for f in sorted(glob.glob('gpurun_out/res1/*_?.json')):
    l=[x for x in open(f).read().splitlines() if x.startswith('{')][-1]; j=json.loads(l)
    print(f, round(j['ms_per_step'],4), round(j['ms_per_step_sync'],4))
PY
