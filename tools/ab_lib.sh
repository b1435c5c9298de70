# A/B of two builds of the same ABI on one box (NKB_LIB selects the library):
#   tools/ab_lib.sh <tag> <ngpus> <config> <rounds>
# alternates prev/new so that box drift hits both; prints ms/step per run.
set -u
TAG=$1; N=$2; CFG=$3; R=${4:-2}
D=gpurun_out/$TAG; mkdir -p $D
L=paper_2312_09888_b200/lib
for r in $(seq 1 $R); do
  for lib in prev new; do
    f=$L/libnekb200.so; [ $lib = prev ] && f=$L/libnekb200_prev.so
    if [ $N = 1 ]; then
      NKB_LIB=$f timeout 600 python bench.py --config $CFG --steps 50 --warmup 5 > $D/${CFG}_${N}_${lib}_$r.json 2> $D/${CFG}_${N}_${lib}_$r.err
    else
      NKB_LIB=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29500+N+r)) bench.py --gpus $N --config $CFG --steps 50 --warmup 5 --e2e-max-gb 0 \
        > $D/${CFG}_${N}_${lib}_$r.json 2> $D/${CFG}_${N}_${lib}_$r.err
    fi
    python -c "import json,sys;d=json.load(open('$D/${CFG}_${N}_${lib}_$r.json'));print('$CFG n=$N $lib r$r', round(d['ms_per_step'],4), d.get('stages_ms'))" || tail -3 $D/${CFG}_${N}_${lib}_$r.err
  done
done
