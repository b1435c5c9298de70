O=gpurun_out/u1e; rm -rf $O; mkdir -p $O
L=paper_2312_09888_b200/lib
for r in 1 2 3 4 5; do
  NKB_LIB=$L/libnekb200_prev.so python tools/kbench.py c5 --reps 20 --tag head >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c5 --reps 20 --tag pre1 >> $O/kb.jsonl 2>> $O/kb.err
done
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw,temperature.gpu --format=csv > $O/smi.txt
python - <<'PY'
import json, collections, statistics
d = collections.defaultdict(list)
for l in open('gpurun_out/u1e/kb.jsonl'):
    j = json.loads(l); d[(j['config'], j['tag'])].append(j['fused'])
for k in sorted(d): print(k, d[k], 'median', statistics.median(d[k]))
PY
cat $O/smi.txt
