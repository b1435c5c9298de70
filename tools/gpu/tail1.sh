# one-GPU resolve tail: GPU suite (product + checked), smoke, bench C2 x2
O=gpurun_out/tail1; rm -rf $O; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so python -m pytest tests -m gpu -q -x > $O/pytest_checked.log 2>&1; echo "checked rc=$?" >> $O/pytest_checked.log; tail -n 2 $O/pytest_checked.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for r in 1 2; do python bench.py --steps 20 --warmup 5 > $O/c2_$r.json 2> $O/c2_$r.err; done
for f in $O/c2_*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4), d['stages_ms'], d['roofline']['frac'], d['parity'], d['e2e']['value']/1e9)"; done
