O=gpurun_out/nvl; rm -rf $O; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 600 python tools/nvlink_probe.py 256 > $O/nvlink_probe.json 2> $O/nvlink_probe.err; echo "rc=$?"
cat $O/nvlink_probe.json; tail -3 $O/nvlink_probe.err
