# bulk composite at 2 stages (64 KB/CTA): overlap vs sequential for C2/C3s/C5 on 4 GPUs; multi tests
O=gpurun_out/ov11; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log; tail -n 2 $O/pytest_multi.log
run() { local n=$1; shift; timeout 600 python bench.py "$@" --no-cpu-baseline --e2e-max-gb 0 > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
for r in 1 2; do
run c2_4_ov_$r --gpus 4 --steps 30 --warmup 5
NKB_COMPOSITE_OVERLAP=0 run c2_4_seq_$r --gpus 4 --steps 30 --warmup 5
run c3s_4_ov_$r --config c3 --scaling strong --gpus 4 --steps 30 --warmup 3
NKB_COMPOSITE_OVERLAP=0 run c3s_4_seq_$r --config c3 --scaling strong --gpus 4 --steps 30 --warmup 3
run c5_4_ov_$r --config c5 --gpus 4 --steps 30 --warmup 3
NKB_COMPOSITE_OVERLAP=0 run c5_4_seq_$r --config c5 --gpus 4 --steps 30 --warmup 3
done
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('ms_per_step_sync',0),4))"; done
