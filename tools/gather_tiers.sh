#!/bin/bash
# k_gather phase time (bench CUDA events) per tier setting on C4 (dev tool):
# GEE_GATHER_MODE 4 = contig, 6 = L1 tiers, 7 = smem head + L1 tiers
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-push 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['roofline']['phases']; print('$*', 'gather %.3f' % p['gather']['ms'], 'step %.3f' % d['ms_per_step'])"
}
run GEE_GATHER_MODE=4
for l1 in 65536 262144 1048576 4194304; do run GEE_GATHER_MODE=6 GEE_GATHER_L1_HOT=$l1; done
for sm in 98304 163840 200704 225280; do
  for l1 in 0 1048576; do run GEE_GATHER_MODE=7 GEE_GATHER_SMEM_HOT=$sm GEE_GATHER_L1_HOT=$l1; done
done
