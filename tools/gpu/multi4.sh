# 4-GPU lease: multi-GPU tests, self-spawning bench at N=2/4 (weak C2), strong C3,
# C5 diagonal, NCCL vs P2P composite, NVLink byte counters around a P2P run
O=gpurun_out/m4; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
run() { # name, args...
  local n=$1; shift
  timeout 900 python bench.py "$@" > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"
}
run c2_1 --steps 20 --warmup 5 --no-cpu-baseline
run c2_2 --gpus 2 --steps 20 --warmup 5
nvidia-smi nvlink -gt d > $O/nvl_before.txt 2>&1
run c2_4 --gpus 4 --steps 200 --warmup 5 --e2e-max-gb 0
nvidia-smi nvlink -gt d > $O/nvl_after.txt 2>&1
NKB_COMPOSITE=nccl run c2_4_nccl --gpus 4 --steps 20 --warmup 5 --e2e-max-gb 0
run c3s_1 --config c3 --scaling strong --steps 10 --warmup 3 --no-cpu-baseline
run c3s_2 --config c3 --scaling strong --gpus 2 --steps 10 --warmup 3 --e2e-max-gb 0
run c3s_4 --config c3 --scaling strong --gpus 4 --steps 10 --warmup 3 --e2e-max-gb 0
run c5_1 --config c5 --steps 10 --warmup 3 --no-cpu-baseline
run c5_2 --config c5 --gpus 2 --steps 10 --warmup 3 --e2e-max-gb 0
run c5_4 --config c5 --gpus 4 --steps 10 --warmup 3 --e2e-max-gb 0
run c4_4 --config c4 --gpus 4 --steps 10 --warmup 3 --e2e-max-gb 0
for f in $O/*.json; do python -c "
import json
t=[l for l in open('$f').read().splitlines() if l.startswith('{')]
d=json.loads(t[-1]) if t else {}
print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), d.get('stages_ms'), d.get('fused_ms_per_rank'))"; done
tail -3 $O/pytest.log
