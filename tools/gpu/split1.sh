# K1g kSplit (C2 at three CTAs per SM): parity + A/B
O=gpurun_out/split1; rm -rf $O; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_checked.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -n 3 $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2 or prog or box" > $O/pytest_checked.log 2>&1; echo "checked rc=$?" >> $O/pytest_checked.log; tail -n 2 $O/pytest_checked.log
for r in 1 2 3; do
  NKB_K1G_SPLIT=0 python tools/kbench.py c2 --reps 30 --tag occ2 >> $O/kb.jsonl 2>> $O/kb.err
  python tools/kbench.py c2 --reps 30 --tag split3 >> $O/kb.jsonl 2>> $O/kb.err
done
cat $O/kb.jsonl
python bench.py --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; python -c "
import json
l=[x for x in open('$O/bench_c2.json').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('bench', round(d['value']/1e9,2), round(d['ms_per_step'],4), d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity']['ok'])"
