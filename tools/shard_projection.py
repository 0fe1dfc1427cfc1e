"""Row-shard step times of C4 at N = 1, 2, 4, 8 shards, measured one shard at
a time on one B200 (dev / profiles tool).

Row-range sharding (shard.build_row_shard) has no
collective in the timed region: each rank runs the histogram of all labels
and the pull of its own rows, and the step's time is the max over ranks.
This box exposes one GPU, so every rank's step is timed here in turn: it
builds that rank's shard, warms it up, and times `--steps` steps with CUDA
events on the launching stream, exactly as bench.py does for each rank. The
projection value = listed edges / max-over-ranks step time assumes that
ranks on separate GPUs do not slow each other down. Nothing crosses NVLink
or PCIe in the timed region, so only the host would be shared.

--scheme edges times the edge-range alternative (SURVEY 8e scheme 2) the
same way: rank r pushes its contiguous slice of the listed edges into a full
fp32 Z partial (zeroed in the step).  The NCCL reduce-scatter that follows
cannot run on one GPU. Its time is modelled from the bytes each rank
contributes, (N-1)/N * n*K*4, at the measured 8-rank bus bandwidth of
725 GB/s (B200_PROFILING.md), and reported separately.

Usage: python tools/shard_projection.py [--shards 1,2,4,8] [--steps 10] [--scheme rows|edges]
Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scheme", default="rows", choices=["rows", "edges"])
    args = ap.parse_args()

    import torch

    from paper_2402_04403_b200 import shard as shard_mod
    from paper_2402_04403_b200 import synth
    from paper_2402_04403_b200.device import DeviceGraph, Embedder

    torch.cuda.set_device(0)
    src, dst, w, y, n, k, _ = synth.make_config(args.config)
    s = int(src.numel())
    cfg = synth.CONFIGS[args.config]
    out = {"workload": cfg.name, "scheme": args.scheme, "s_listed_edges": s, "steps": args.steps,
           "warmup": args.warmup, "per_n": {}}
    BUS_GBS = 725.0
    ALLREDUCE_MS = 0.025  # NCCL all-reduce of k+1 int64 over NVLink: latency-bound, ~25 us
    for nshards in (int(x) for x in args.shards.split(",")):
        ranks = []
        for rank in range(nshards):
            if args.scheme == "edges":
                e = shard_mod.plan_edges(s, nshards)
                e0, e1 = int(e[rank]), int(e[rank + 1])
                g = DeviceGraph.from_edges(src[e0:e1], dst[e0:e1], None if w is None else w[e0:e1], n, pull=False)
                emb = Embedder(n, k)
                z = torch.empty((n, k), dtype=torch.float32, device="cuda")
                emb.project(y, validate=True)
                run = lambda: (emb.project(y, validate=False), emb.push(g, z))  # noqa: E731
                for _ in range(args.warmup):
                    run()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(args.steps):
                    run()
                b.record()
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / args.steps
                rs_bytes = (nshards - 1) / nshards * n * k * 4
                ranks.append({"rank": rank, "edges": e1 - e0, "ms_per_step": ms, "reduce_scatter_bytes": rs_bytes,
                              "reduce_scatter_ms_model": rs_bytes / (BUS_GBS * 1e9) * 1e3})
                del g, emb, z
                torch.cuda.empty_cache()
                continue
            if nshards == 1:
                g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
                lo, hi = 0, n
            else:
                g, lo, hi = shard_mod.build_row_shard(src, dst, w, n, nshards, rank, k=k)
            g.prepare_hot(k)
            g.tile_heavy()
            emb = Embedder(n, k)
            z = torch.empty((hi - lo, k), dtype=torch.float32, device="cuda")
            emb.project(y, validate=True, g=g)
            # as bench.py: with several ranks the histogram is sharded (each
            # rank counts n/N labels; the all-reduce of k+1 counts is modelled)
            c_lo, c_hi = shard_mod.label_slice(n, nshards, rank)

            def proj():
                if nshards > 1:
                    emb.project_sharded(y, g, c_lo, c_hi, lambda c: c)
                else:
                    emb.project(y, validate=False, g=g)

            for _ in range(args.warmup):
                proj()
                emb.pull(g, z)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.steps):
                proj()
                emb.pull(g, z)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / args.steps
            ranks.append({"rank": rank, "rows": hi - lo, "arcs": int(g.arcs), "ms_per_step": ms,
                          "allreduce_ms_model": ALLREDUCE_MS if nshards > 1 else 0.0})
            del g, emb, z
            torch.cuda.empty_cache()
        worst = max(r["ms_per_step"] + r.get("reduce_scatter_ms_model", 0.0) + r.get("allreduce_ms_model", 0.0)
                    for r in ranks)
        mean = sum(r["ms_per_step"] for r in ranks) / len(ranks)
        out["per_n"][nshards] = {"max_ms": worst, "mean_ms": mean, "balance": mean / worst,
                                 "projected_geps": s / (worst * 1e-3) / 1e9, "ranks": ranks}
    base = out["per_n"].get(1)
    if base:
        for nshards, r in out["per_n"].items():
            r["projected_efficiency"] = base["max_ms"] / (nshards * r["max_ms"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
