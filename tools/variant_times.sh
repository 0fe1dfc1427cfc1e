#!/bin/bash
# per-variant launch times of one kernel (ncu launch list; dev tool)
# usage: tools/variant_times.sh <kernel-regex> <variant>...   ("" = default lib)
kre=$1; shift
for v in "$@"; do
  GEE_LIB_VARIANT=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$kre" -c 2 --csv \
    --log-file gpurun_out/vt_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-push > /dev/null 2>&1
  echo "variant=$v $(grep -v '^==' gpurun_out/vt_$v.csv | tail -n +2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
