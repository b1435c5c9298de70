O=gpurun_out/m4head; rm -rf $O; mkdir -p $O
run() { local n=$1; shift; timeout 600 python bench.py "$@" --no-cpu-baseline --e2e-max-gb 0 > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
run c2_4 --gpus 4 --steps 30 --warmup 5
run c3s_1 --config c3 --scaling strong --steps 20 --warmup 3
run c3s_4 --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3
run c5_4 --config c5 --gpus 4 --steps 20 --warmup 3
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), d.get('composite_overlapped'))"; done
