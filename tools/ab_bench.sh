#!/bin/bash
# dev tool (GPU box): C4 device-resident step for each extra bench.py flag set given as an argument
for f in "$@"; do
  timeout 400 python bench.py --no-e2e --no-cpu --no-push $f > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('[$f]', round(d['ms_per_step'],3), round(d['value'],2), {k:round(v['ms'],3) for k,v in d['roofline']['phases'].items()}, d['config'].get('scale_exp'), d['config'].get('qmax'))
"
done
