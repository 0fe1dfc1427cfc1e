#!/bin/bash
# k_gather phase time (bench CUDA events) per head setting on C4 (dev tool):
# GEE_GATHER_MODE 4 = contig, 6 = L1 tiers, 7 = smem head + L1 tiers,
# 8 / 9 = byte head + one load (L1 default / evict_last), 10 = packed head
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-push 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['roofline']['phases']; print('$*', 'gather %.3f' % p['gather']['ms'], 'step %.3f' % d['ms_per_step'])"
}
for bt in ${BLOCKS:-512 768 1024}; do
  for sm in ${SMEMS:-98304 131072 163840 196608}; do run GEE_GATHER_BLOCK=$bt GEE_GATHER_SMEM_HOT=$sm; done
done
