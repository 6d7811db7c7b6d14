#!/bin/bash
# C3 batch: lanes A/B after the session-5 kernel changes
mkdir -p gpurun_out
for nl in 1 2 3 4; do
  timeout 900 python bench.py --workload c3 --steps 1 --warmup 3 --lanes $nl --no-cpu-baseline > gpurun_out/s5_c3_l$nl.json 2> gpurun_out/s5_c3_l$nl.err
  python -c "import json;d=json.loads([l for l in open('gpurun_out/s5_c3_l$nl.json') if l.startswith('{')][-1]);print('lanes',$nl,'value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"
done
