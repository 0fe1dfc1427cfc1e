#!/bin/bash
# k_gather time per (GEE_GATHER_MODE, GEE_GATHER_SMEM_HOT) on C4 (dev tool)
for mode in ${MODES:-0 1 2 3}; do
  for sm in ${SMEMS:-0 32768 65536 131072}; do
    GEE_GATHER_MODE=$mode GEE_GATHER_SMEM_HOT=$sm ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct --clock-control none \
      -k regex:k_gather -s 2 -c 1 --csv --log-file gpurun_out/gs.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-push > /dev/null 2>&1
    echo "mode=$mode smem=$sm $(grep -v '^==' gpurun_out/gs.csv | tail -n +2 | awk -F'","' '{print $(NF-2)":"$NF}' | tr -d '"' | tr '\n' ' ')"
  done
done
