"""Run bench.py with a watchdog (dev tool): after 150 s every thread's Python
stack is dumped and the process exits.  Under torchrun this shows where each
rank of a hung multi-rank run is waiting, e.g.
    GEE_BENCH_BACKEND=gloo python -m torch.distributed.run --nproc-per-node 2 \
        --master-addr 127.0.0.1 tools/fh_bench.py --gpus 2 --scale 22 --no-e2e --no-cpu
"""
import faulthandler
import runpy
import sys

faulthandler.dump_traceback_later(150, exit=True)
sys.argv = ["bench.py"] + sys.argv[1:]
runpy.run_path("bench.py", run_name="__main__")
