set -u
D=gpurun_out/s2/multi; mkdir -p $D
nvidia-smi topo -m > $D/topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stats.py tests/test_gpu_dssum.py -q -x > $D/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -2 $D/pytest_multi.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) \
    bench.py --gpus $n --steps 20 --warmup 5 > $D/c2_$n.json 2> $D/c2_$n.err; echo "c2 n=$n rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 \
  bench.py --gpus 4 --steps 10 --warmup 3 --config c4 --e2e-max-gb 4 > $D/c4_4.json 2> $D/c4_4.err; echo "c4 n=4 rc=$?"
