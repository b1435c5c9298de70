O=gpurun_out/ov6; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_partitions.py -m gpu -q -x > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log
tail -n 3 $O/pytest_multi.log
for n in 2 4; do
B="timeout 300 python bench.py --gpus $n --steps 50 --warmup 5 --no-cpu-baseline --e2e-max-gb 0"
for r in 1 2 3; do
  $B > $O/c2_${n}_on4_$r.json 2> $O/c2_${n}_on4_$r.err
  NKB_COMPOSITE_SMS=8 $B > $O/c2_${n}_on8_$r.json 2> $O/c2_${n}_on8_$r.err
  NKB_COMPOSITE_OVERLAP=0 $B > $O/c2_${n}_off_$r.json 2> $O/c2_${n}_off_$r.err
done
done
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/c2_1.json 2> $O/c2_1.err
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4), round(d['host_ms_per_async_launch'],4), d['stages_ms'])"; done
