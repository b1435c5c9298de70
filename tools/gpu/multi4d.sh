# final 4-GPU set: full GPU suite, C2 weak 1/2/4 (P2P and NCCL), C3 strong 1/2/4, C5 weak 1/2/4, C4 4
O=gpurun_out/m4d; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
run() { local n=$1; shift; timeout 900 python bench.py "$@" > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
run c2_1 --steps 50 --warmup 5 --no-cpu-baseline
run c2_2 --gpus 2 --steps 50 --warmup 5 --e2e-max-gb 0
run c2_4 --gpus 4 --steps 50 --warmup 5 --e2e-max-gb 0
NKB_COMPOSITE_OVERLAP=0 run c2_4_seq --gpus 4 --steps 50 --warmup 5 --e2e-max-gb 0
NKB_COMPOSITE=nccl run c2_4_nccl --gpus 4 --steps 50 --warmup 5 --e2e-max-gb 0
run c3s_1 --config c3 --scaling strong --steps 20 --warmup 3 --no-cpu-baseline
run c3s_2 --config c3 --scaling strong --gpus 2 --steps 20 --warmup 3 --e2e-max-gb 0
run c3s_4 --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3 --e2e-max-gb 0
NKB_COMPOSITE_OVERLAP=0 run c3s_4_seq --config c3 --scaling strong --gpus 4 --steps 20 --warmup 3 --e2e-max-gb 0
run c5_1 --config c5 --steps 20 --warmup 3 --no-cpu-baseline
run c5_2 --config c5 --gpus 2 --steps 20 --warmup 3 --e2e-max-gb 0
run c5_4 --config c5 --gpus 4 --steps 20 --warmup 3 --e2e-max-gb 0
run c4_1 --config c4 --steps 10 --warmup 3 --no-cpu-baseline
run c4_4 --config c4 --gpus 4 --steps 10 --warmup 3 --e2e-max-gb 0
run c4_4_work --config c4 --gpus 4 --steps 10 --warmup 3 --e2e-max-gb 0 --partition work
tail -3 $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_partitions.py -m gpu -q > $O/pytest_checked_multi.log 2>&1; echo "checked rc=$?" >> $O/pytest_checked_multi.log
tail -3 $O/pytest_checked_multi.log
for f in $O/c*.json; do python -c "
import json
l=[x for x in open('$f').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('$f', d['n_gpus'], round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('ms_per_step_sync',0),4), d['stages_ms'].get('composite'), d.get('fused_ms_per_rank'))"; done
