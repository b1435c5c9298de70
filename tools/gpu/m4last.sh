O=gpurun_out/m4last; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_multi.py tests/test_gpu_partitions.py tests/test_gpu_dssum.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
run() { local n=$1; shift; timeout 600 python bench.py "$@" --no-cpu-baseline --e2e-max-gb 0 > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
run c2_1 --steps 30 --warmup 5
run c2_2 --gpus 2 --steps 30 --warmup 5
run c2_4 --gpus 4 --steps 30 --warmup 5
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), d.get('composite_overlapped'), d.get('gpu_launches'))"; done
