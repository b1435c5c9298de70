O=gpurun_out/ov10; rm -rf $O; mkdir -p $O
for cfg in c5 c3; do
  extra=""; [ $cfg = c3 ] && extra="--scaling strong"
  NKB_SPLIT_TRACE=1 timeout 300 python bench.py --config $cfg $extra --gpus 4 --steps 20 --warmup 3 --no-cpu-baseline --e2e-max-gb 0 > $O/$cfg.json 2> $O/$cfg.err
  python -c "
import json
l=[x for x in open('$O/$cfg.json').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$cfg', round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4), d['stages_ms'], d['fused_ms_per_rank'])"
  for r in 0 1 2 3; do grep "rank $r\]" $O/$cfg.err | tail -21 | sed -n '8,11p' | cut -c1-110; done
  NKB_COMPOSITE_OVERLAP=0 timeout 300 python bench.py --config $cfg $extra --gpus 4 --steps 20 --warmup 3 --no-cpu-baseline --e2e-max-gb 0 > $O/${cfg}_seq.json 2> $O/${cfg}_seq.err
  python -c "
import json
l=[x for x in open('$O/${cfg}_seq.json').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$cfg seq', round(d['ms_per_step'],4), round(d['ms_per_step_sync'],4))"
done
