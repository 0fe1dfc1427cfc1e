# dev tool (GPU box): streamed e2e by the number of host expansion threads (HostPipeline.EXPAND_THREADS_STREAMED)
for t in 6 8 10 12; do
python - <<PY > gpurun_out/s9_thr.json 2>/dev/null
import sys, runpy
from paper_2402_04403_b200.stream import HostPipeline
HostPipeline.EXPAND_THREADS_STREAMED = $t
sys.argv = ["bench.py", "--no-cpu", "--no-push", "--no-e2e-resident", "--e2e-steps", "5"]
runpy.run_path("bench.py", run_name="__main__")
PY
python -c "
import json
d=json.loads(open('gpurun_out/s9_thr.json').read().strip().splitlines()[-1])
print($t, round(d['e2e']['ms_per_step'],1), round(d['e2e']['value'],3), d['e2e']['chunks'])
"
done
