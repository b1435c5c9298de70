O=gpurun_out/fork; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for r in 1 2 3; do python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/c2_$r.json 2> $O/c2_$r.err; done
for f in $O/c2_*.json; do python -c "
import json; d=json.load(open('$f')); print(d['ms_per_step'], d['ms_per_step_sync'], d['stages_ms'])"; done
tail -2 $O/pytest.log
