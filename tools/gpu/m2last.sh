O=gpurun_out/m2last; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_multi.py tests/test_gpu_partitions.py tests/test_gpu_dssum.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
for n in 1 2; do python bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/c2_$n.json 2> $O/c2_$n.err; done
for f in $O/c2_*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), d.get('composite_overlapped'), d['gpu_launches'])"; done
