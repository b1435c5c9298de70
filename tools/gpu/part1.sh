# C4 / C3 on 4 GPUs: equal contiguous ranges vs work-balanced contiguous ranges
O=gpurun_out/part1; rm -rf $O; mkdir -p $O
run() { local n=$1; shift; timeout 900 python bench.py "$@" > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
run c4_4_equal --config c4 --gpus 4 --steps 20 --warmup 3 --e2e-max-gb 0 --no-cpu-baseline
run c4_4_work --config c4 --gpus 4 --steps 20 --warmup 3 --e2e-max-gb 0 --no-cpu-baseline --partition work
run c4_2_work --config c4 --gpus 2 --steps 20 --warmup 3 --e2e-max-gb 0 --no-cpu-baseline --partition work
run c4_2_equal --config c4 --gpus 2 --steps 20 --warmup 3 --e2e-max-gb 0 --no-cpu-baseline
run c4_1 --config c4 --steps 20 --warmup 3 --e2e-max-gb 0 --no-cpu-baseline
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('ms_per_step_sync',0),4), d['stages_ms'], d.get('fused_ms_per_rank'), d.get('triangles_per_rank'), (d['config'].get('partition') or {}).get('cuts'))"; done
tail -3 $O/c4_4_work.err
