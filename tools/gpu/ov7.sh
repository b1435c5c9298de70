O=gpurun_out/ov7; rm -rf $O; mkdir -p $O
for sms in 4 16; do
NKB_SPLIT_TRACE=1 NKB_COMPOSITE_SMS=$sms timeout 300 python bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline --e2e-max-gb 0 > $O/t$sms.json 2> $O/t$sms.err
python -c "
import json
l=[x for x in open('$O/t$sms.json').read().splitlines() if x.startswith('{')][-1]
d=json.loads(l);print('sms $sms', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['host_ms_per_async_launch'],4))"
for r in 0 1 2 3; do grep "rank $r\]" $O/t$sms.err | grep -v "step 0 " | sed -n '10,14p'; done
done
