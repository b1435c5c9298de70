set -u
mkdir -p gpurun_out/r03_scaling
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r03_scaling/c2_$n.json 2> gpurun_out/r03_scaling/c2_$n.err
  echo "n=$n rc=$?"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 4 --steps 10 --warmup 3 --config c4 --e2e-max-gb 4 > gpurun_out/r03_scaling/c4_4.json 2> gpurun_out/r03_scaling/c4_4.err
echo "c4 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r03_scaling/ref_1.json 2> gpurun_out/r03_scaling/ref_1.err
echo "ref rc=$?"
for f in gpurun_out/r03_scaling/*.json; do echo $f; python -c "
import json,sys
t=[l for l in open('$f').read().splitlines() if l.startswith('{')]
d=json.loads(t[-1]) if t else {}
print(d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), d.get('stages_ms'), d.get('fused_ms_per_rank'))"; done
