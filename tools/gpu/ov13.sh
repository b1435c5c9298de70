# overlap policy (<= 2 CTAs/SM surface passes) + device-barrier start: 4-GPU lines; multi tests
O=gpurun_out/ov13; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log; tail -n 2 $O/pytest_multi.log
run() { local n=$1; shift; timeout 600 python bench.py "$@" --no-cpu-baseline --e2e-max-gb 0 > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
for r in 1 2; do
run c2_4_$r --gpus 4 --steps 20 --warmup 5
run c3s_4_$r --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3
run c4_4_$r --config c4 --gpus 4 --steps 10 --warmup 3
NKB_COMPOSITE_OVERLAP=0 run c4_4_seq_$r --config c4 --gpus 4 --steps 10 --warmup 3
run c4_4_work_$r --config c4 --gpus 4 --steps 10 --warmup 3 --partition work
done
run c5_4 --config c5 --gpus 4 --steps 20 --warmup 3
run c2_2 --gpus 2 --steps 20 --warmup 5
run c2_1 --steps 20 --warmup 5
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('ms_per_step_sync',0),4), d.get('composite_overlapped'), d.get('gpu_launches'))"; done
