# dev tool: C4 device-resident step against the tile count / tile size of the heavy region
# usage: bash tools/tile_sweep.sh 21:196608 42:196608 ...
for cfg in "$@"; do T=${cfg%%:*}; S=${cfg##*:}
timeout 400 python bench.py --no-e2e --no-cpu --no-push --heavy-layout tiles --tile-max $T --tile-slots $S > gpurun_out/tl_${T}_$S.json 2> gpurun_out/tl_${T}_$S.err; tail -2 gpurun_out/tl_${T}_$S.err
python -c "
import json,sys
d=json.loads(open('gpurun_out/tl_${T}_$S.json').read().strip().splitlines()[-1])
print('T=$T ts=$S', round(d['ms_per_step'],3), {k:round(v['ms'],3) for k,v in d['roofline']['phases'].items()}, d['config']['padded_arcs'], d['config'].get('l2_path_arcs'))
"; done
