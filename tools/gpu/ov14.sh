# forced overlap beside 3-CTA K1g (C3 strong, C5 weak) with the device-barrier start: stability check
O=gpurun_out/ov14; rm -rf $O; mkdir -p $O
run() { local n=$1; shift; timeout 600 python bench.py "$@" --no-cpu-baseline --e2e-max-gb 0 > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
for r in 1 2 3; do
NKB_COMPOSITE_OVERLAP=2 run c3s_4_ov2_$r --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3
NKB_COMPOSITE_OVERLAP=2 NKB_COMPOSITE_SMS=8 run c3s_4_ov2s8_$r --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3
run c3s_4_seq_$r --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3
done
for r in 1 2; do
NKB_COMPOSITE_OVERLAP=2 run c5_4_ov2_$r --config c5 --gpus 4 --steps 20 --warmup 3
run c5_4_seq_$r --config c5 --gpus 4 --steps 20 --warmup 3
done
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', round(d['ms_per_step'],4), d.get('composite_overlapped'))"; done
