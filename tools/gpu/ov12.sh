# device barrier before the start event: run-to-run spread of 4-GPU lines (overlap vs sequential)
O=gpurun_out/ov12; rm -rf $O; mkdir -p $O
run() { local n=$1; shift; timeout 600 python bench.py "$@" --no-cpu-baseline --e2e-max-gb 0 > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
for r in 1 2 3; do
run c2_4_ov_$r --gpus 4 --steps 20 --warmup 5
NKB_COMPOSITE_OVERLAP=0 run c2_4_seq_$r --gpus 4 --steps 20 --warmup 5
run c3s_4_ov_$r --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3
NKB_COMPOSITE_OVERLAP=0 run c3s_4_seq_$r --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3
done
run c2_1 --steps 20 --warmup 5
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('ms_per_step_sync',0),4))"; done
tail -3 $O/c2_4_ov_1.err
