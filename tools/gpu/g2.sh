O=gpurun_out/g2; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py --steps 20 --warmup 5 > $O/c2_1.json 2> $O/c2_1.err; echo "c2_1 rc=$?"
python bench.py --gpus 2 --steps 20 --warmup 5 > $O/c2_2.json 2> $O/c2_2.err; echo "c2_2 rc=$?"
python bench.py --config c5 --gpus 2 --steps 10 --warmup 3 --e2e-max-gb 0 > $O/c5_2.json 2> $O/c5_2.err; echo "c5_2 rc=$?"
tail -2 $O/pytest.log
for f in $O/c*.json; do python -c "
import json
d=json.load(open('$f'));print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4), d['stages_ms'], (d.get('parity') or {}).get('ok'))"; done
