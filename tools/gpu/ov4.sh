O=gpurun_out/ov4; rm -rf $O; mkdir -p $O
B="timeout 300 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-max-gb 0"
NKB_SPLIT_TRACE=1 $B > $O/c2_on2.json 2> $O/c2_on2.err
NKB_SPLIT_TRACE=1 NKB_COMPOSITE_SMS=0 $B > $O/c2_on0.json 2> $O/c2_on0.err
grep "nkb split" $O/c2_on2.err | head -60 > $O/trace_on2.txt
grep "nkb split" $O/c2_on0.err | head -60 > $O/trace_on0.txt
head -30 $O/trace_on2.txt; head -30 $O/trace_on0.txt
