# 1-GPU C5 sweep: the six BASELINE configs[4] sizes
O=gpurun_out/c5; mkdir -p $O
for E in 65536 131072 262144 524288 1048576 2097152; do
  timeout 900 python bench.py --config c5 --elements $E --steps 10 --warmup 3 --csv $O/csv_$E > $O/c5_$E.json 2> $O/c5_$E.err
  echo "E=$E rc=$?"
done
for f in $O/c5_*.json; do python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f', d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d['stages_ms'], d.get('parity',{}).get('ok'))"; done
