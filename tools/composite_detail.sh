OUT=${1:-r09ab3}
mkdir -p gpurun_out/$OUT
L=paper_2312_09888_b200/lib
for lib in prev new; do
  f=$L/libnekb200.so; [ $lib = prev ] && f=$L/libnekb200_prev.so
  NKB_TIMING_DETAIL=1 NKB_LIB=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 4 --config c2 --steps 20 --warmup 5 --e2e-max-gb 0 > gpurun_out/$OUT/detail_$lib.json 2> gpurun_out/$OUT/detail_$lib.err
  echo "$lib composite kernel (median over lines):"; grep "nkb composite" gpurun_out/$OUT/detail_$lib.err | awk '{print $7}' | sort -n | awk '{a[NR]=$1} END {print "n="NR, "median", a[int(NR/2)+1], "p90", a[int(NR*0.9)]}'
done
