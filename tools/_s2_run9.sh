set -u
D=gpurun_out/s2/m2; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > $D/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -2 $D/pytest_multi.log
for i in 1 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $D/c2_2_$i.json 2> $D/c2_2_$i.err; echo "c2 n=2 rc=$?"
NKB_COMPOSITE=nccl timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29503 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $D/c2_2_nccl_$i.json 2> $D/c2_2_nccl_$i.err; echo "c2 n=2 nccl rc=$?"
done
timeout 600 python tools/gpu_probe.py c1 --reps 3 --device-gen --geo on > $D/c1_probe.log 2>&1; echo "c1 probe rc=$?"
timeout 600 python tools/gpu_probe.py c2 --reps 3 --device-gen --geo on > $D/c2_probe.log 2>&1; echo "c2 probe rc=$?"
grep "rep 2" $D/c1_probe.log $D/c2_probe.log
