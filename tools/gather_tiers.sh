#!/bin/bash
# k_gather phase time (bench CUDA events) per tier setting on C4 (dev tool):
# GEE_GATHER_MODE 4 = contig, 6 = L1 tiers, 7 = smem head + L1 tiers,
# 8 / 9 = smem head + one load (L1 default / evict_last)
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-push 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['roofline']['phases']; print('$*', 'gather %.3f' % p['gather']['ms'], 'step %.3f' % d['ms_per_step'])"
}
run GEE_GATHER_MODE=4
for m in ${MODES:-9}; do
  for sm in ${SMEMS:-81920 90112 98304 106496 114688}; do run GEE_GATHER_MODE=$m GEE_GATHER_SMEM_HOT=$sm; done
done
