#!/bin/bash
# time the pull with phases skipped (experiment; results wrong when skipping)
for sk in ${@:-0 15 31 63}; do
  echo -n "skip=$sk "; GEE_PULL_VERBOSE=1 GEE_PULL_SKIP=$sk timeout 300 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu --no-push 2>gpurun_out/skip_$sk.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'ms', round(d['roofline']['pull_ms'],2))"; grep -m1 k_pull gpurun_out/skip_$sk.err
done
