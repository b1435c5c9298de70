# final 1-GPU set at HEAD: smoke, GPU suite (product + checked), bench per config, reference arm
O=gpurun_out/final7; rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
NKB_LIB=paper_2312_09888_b200/lib/libnekb200_checked.so python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_checked.log 2>&1; echo "pytest(checked) rc=$?" >> $O/pytest_checked.log
python bench.py --steps 20 --warmup 5 --csv $O/csv_c2 > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_c2.json 2> $O/ref_c2.err; echo "ref rc=$?"
python bench.py --config c1 --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1 rc=$?"
python bench.py --config c3 --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python bench.py --config c4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
python bench.py --config c5 --steps 10 --warmup 3 > $O/c5_65536.json 2> $O/c5_65536.err; echo "c5 rc=$?"
for f in $O/smoke.log $O/pytest.log $O/pytest_checked.log; do tail -n 2 $f; done
python tools/tables.py $O
