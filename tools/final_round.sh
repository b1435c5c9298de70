# Final measurement set of a round (run on a 4-GPU box via gpurun --gpus 4):
# 1-GPU bench lines for every config, 2/4-GPU weak scaling of C2, C4 on 4
# GPUs, and the reference arm.  Outputs: gpurun_out/<tag>/*.json
set -u
TAG=${1:-r06}
D=gpurun_out/$TAG
mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stats.py tests/test_gpu_dssum.py -q -x > $D/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -1 $D/pytest_multi.log
for c in c1 c2 c3 c4; do
  python bench.py --config $c --steps 20 --warmup 5 > $D/${c}_1.json 2> $D/${c}_1.err; echo "$c n=1 rc=$?"
done
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) \
    bench.py --gpus $n --steps 20 --warmup 5 > $D/c2_$n.json 2> $D/c2_$n.err; echo "c2 n=$n rc=$?"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 \
  bench.py --gpus 4 --steps 10 --warmup 3 --config c4 --e2e-max-gb 4 > $D/c4_4.json 2> $D/c4_4.err; echo "c4 n=4 rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29700 \
  bench.py --gpus 4 --steps 10 --warmup 3 --config c3 --e2e-max-gb 4 > $D/c3_4.json 2> $D/c3_4.err; echo "c3 n=4 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $D/ref_1.json 2> $D/ref_1.err; echo "ref rc=$?"
