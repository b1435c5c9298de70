O=gpurun_out/pd; mkdir -p $O
python -m pytest tests/test_gpu_dssum.py -q -x > $O/pytest_dssum.log 2>&1; echo "rc=$?" >> $O/pytest_dssum.log; tail -n 3 $O/pytest_dssum.log
python tools/dssum_probe.py 20 > $O/probe.json 2> $O/probe.err && cat $O/probe.json && \
ncu --set full --clock-control none --import-source on -k regex:gs_ -c 3 -f -o $O/dssum python tools/dssum_probe.py 1 > $O/ncu.log 2>&1
echo "ncu rc=$?"
