#!/bin/bash
# k_gather phase time (bench CUDA events) per shared-memory head size on C4
# (dev tool; GEE_GATHER_SMEM_HOT=0: no head)
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-push 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['roofline']['phases']; print('$*', 'gather %.3f' % p['gather']['ms'], 'step %.3f' % d['ms_per_step'])"
}
for sm in ${SMEMS:-0 65536 98304 131072}; do run GEE_GATHER_SMEM_HOT=$sm; done
