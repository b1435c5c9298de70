# round-2 check: GPU suite, bench (compact geometry default vs full layout), reference arm
O=gpurun_out/r1; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py --steps 20 --warmup 5 --csv $O/csv > $O/bench.json 2> $O/bench.err
NKB_GEOM_CACHE=full python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_full.json 2> $O/bench_full.err
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --impl reference --steps 5 --warmup 3 > $O/ref.json 2> $O/ref.err
tail -3 $O/pytest.log; tail -3 $O/bench.err
