O=gpurun_out/nomemset; rm -rf $O; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
for r in 1 2; do python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/c2_$r.json 2> $O/c2_$r.err; done
python bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/c2_4.json 2> $O/c2_4.err
for f in $O/c2_*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('ms_per_step_sync',0),4))"; done
