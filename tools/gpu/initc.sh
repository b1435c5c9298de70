O=gpurun_out/initc; rm -rf $O; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
L=paper_2312_09888_b200/lib
for r in 1 2 3; do
  NKB_LIB=$L/libnekb200_prev.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/head_$r.json 2>/dev/null
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/new_$r.json 2>/dev/null
done
for f in $O/*_?.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4))"; done
