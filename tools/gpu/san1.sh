# K1s block-size A/B, then compute-sanitizer memcheck over every hot-path kernel
O=gpurun_out/san1; mkdir -p $O
for r in 1 2; do for t in 768 896 1024; do
  NKB_STREAM_THREADS=$t python tools/kbench.py c4 --reps 20 --tag t$t >> $O/kb.jsonl 2>> $O/kb.err
done; done
cat $O/kb.jsonl
python tools/sanitize_case.py > $O/plain.log 2>&1 && \
compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_case.py > $O/memcheck.log 2>&1
echo "memcheck rc=$?"; tail -5 $O/memcheck.log
