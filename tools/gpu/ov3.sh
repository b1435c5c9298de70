# bulk composite on 1 GPU (partitions) first, then 2 GPUs: multi tests + bench
O=gpurun_out/ov3; rm -rf $O; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_partitions.py -q -x > $O/pytest_part.log 2>&1; echo "part rc=$?" >> $O/pytest_part.log
tail -n 3 $O/pytest_part.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log
tail -n 3 $O/pytest_multi.log
B="timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-max-gb 0"
for r in 1 2; do
  $B > $O/c2_on2_$r.json 2> $O/c2_on2_$r.err
  NKB_COMPOSITE_SMS=4 $B > $O/c2_on4_$r.json 2> $O/c2_on4_$r.err
  NKB_COMPOSITE_SMS=8 $B > $O/c2_on8_$r.json 2> $O/c2_on8_$r.err
  NKB_COMPOSITE_OVERLAP=0 $B > $O/c2_off_$r.json 2> $O/c2_off_$r.err
done
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4), d['stages_ms'])"; done
