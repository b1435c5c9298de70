O=gpurun_out/c5sweep2; rm -rf $O; mkdir -p $O
for E in 65536 131072 262144 524288 1048576 2097152; do
  timeout 900 python bench.py --config c5 --elements $E --steps 10 --warmup 3 > $O/c5_$E.json 2> $O/c5_$E.err; echo "c5 $E rc=$?"
done
python tools/tables.py $O
