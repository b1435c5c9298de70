O=gpurun_out/refn; rm -rf $O; mkdir -p $O
timeout 600 python bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/ref_2.json 2> $O/ref_2.err; echo "ref2 rc=$?"
tail -c 600 $O/ref_2.json
