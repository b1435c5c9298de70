O=gpurun_out/m2final2; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_multi.py tests/test_gpu_partitions.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so python -m pytest tests/test_gpu_multi.py -m gpu -q > $O/pytest_checked.log 2>&1; echo "checked rc=$?" >> $O/pytest_checked.log; tail -n 2 $O/pytest_checked.log
for n in 1 2; do python bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/c2_$n.json 2> $O/c2_$n.err; done
for f in $O/c2_*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('ms_per_step_sync',0),4), d.get('composite_overlapped'))"; done
