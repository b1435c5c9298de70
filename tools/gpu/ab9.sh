# one-pass DSSUM: GPU tests, then bench next_rows with one- and two-pass DSSUM
O=gpurun_out/ab9; mkdir -p $O
python -m pytest tests/test_gpu_dssum.py tests/test_gpu_multi.py -q -x > $O/pytest_dssum.log 2>&1; echo "rc=$?" >> $O/pytest_dssum.log
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_one.json 2> $O/bench_one.err
NKB_DSSUM_TWO_PASS=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_two.json 2> $O/bench_two.err
tail -2 $O/pytest_dssum.log $O/pytest.log
for f in one two; do python -c "
import json,sys
l=[x for x in open('$O/bench_$f.json').read().splitlines() if x.startswith('{')][-1]
j=json.loads(l); print('$f', json.dumps(j['next_rows']['dssum']))"; done
