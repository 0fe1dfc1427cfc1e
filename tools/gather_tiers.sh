#!/bin/bash
# k_gather phase time (bench CUDA events) per head setting on C4 (dev tool):
# GEE_GATHER_MODE 4 = contig, 6 = L1 tiers, 7 = smem head + L1 tiers,
# 8 / 9 = byte head + one load (L1 default / evict_last), 10 = packed head
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-push 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['roofline']['phases']; print('$*', 'gather %.3f' % p['gather']['ms'], 'step %.3f' % d['ms_per_step'])"
}
run GEE_GATHER_MODE=9
for m in ${MODES:-10}; do
  for sm in ${SMEMS:-65536 81920 98304 114688 131072}; do run GEE_GATHER_MODE=$m GEE_GATHER_SMEM_HOT=$sm; done
done
