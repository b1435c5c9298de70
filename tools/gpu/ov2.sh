# composite overlap (split P2P steps) on 2 GPUs: multi-GPU tests, bench C2 on/off and reserved SMs
O=gpurun_out/ov2; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
B="python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-max-gb 0"
for r in 1 2; do
  $B > $O/c2_on2_$r.json 2> $O/c2_on2_$r.err
  NKB_COMPOSITE_SMS=4 $B > $O/c2_on4_$r.json 2> $O/c2_on4_$r.err
  NKB_COMPOSITE_SMS=0 $B > $O/c2_on0_$r.json 2> $O/c2_on0_$r.err
  NKB_COMPOSITE_OVERLAP=0 $B > $O/c2_off_$r.json 2> $O/c2_off_$r.err
done
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4), d['stages_ms'])"; done
