#!/bin/bash
# dev tool (run on the GPU box): rebuild one CUDA source with -D flags, relink, time the C4 step.
# usage: tools/variant_sweep.sh gee_reduce.cu "-DGEE_RING_H=2 -DGEE_HSUB=2" "-DGEE_RING_H=4 -DGEE_HSUB=2" ...
src=$1; shift
pkg=paper_2402_04403_b200
for flags in "$@" ""; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags -c -o $pkg/build/$src.o $pkg/csrc/$src || exit 1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $pkg/libgee_b200.so $pkg/build/*.cu.o || exit 1
  timeout 400 python bench.py --no-e2e --no-cpu --no-push ${BENCH_ARGS} > gpurun_out/vs.json 2> gpurun_out/vs.err || tail -3 gpurun_out/vs.err
  python -c "
import json
d=json.loads(open('gpurun_out/vs.json').read().strip().splitlines()[-1])
print('flags=[$flags]', round(d['ms_per_step'],3), {k:round(v['ms'],3) for k,v in d['roofline']['phases'].items()})
"
done
