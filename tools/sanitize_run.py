"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every product kernel family once, checked against the CPU oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Covers: histogram + label table (plain and compact hot tier), the packed-head
gather, the block ring reducer and the heavy items (weighted and unit),
the wide reducer (K > 255, light rows and a heavy row), the push (with and
without pre-combine), graph preparation (CSR build, hot plan, row sort and
pad), and the host-streamed pass (pack / unpack targets, Z compaction).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402
from paper_2402_04403_b200.stream import HostPipeline, pinned_like  # noqa: E402


def check(z, exp, what):
    z = z.cpu().numpy() if isinstance(z, torch.Tensor) else z
    nz = exp != 0
    assert np.all(z[~nz] == 0), what
    err = float(np.max(np.abs(z[nz] - exp[nz]) / np.abs(exp[nz]))) if nz.any() else 0.0
    assert err <= 1e-4, (what, err)
    print(f"{what}: ok (max rel err {err:.1e})", flush=True)


def main():
    dev = torch.device("cuda")
    scale, s = 15, 200_000
    n = 1 << scale
    for weighted, k in ((True, 50), (False, 7)):
        src, dst, w = synth.rmat_edges(scale, s, seed=3, weighted=weighted, device=dev)
        # one hub row above the heavy threshold (2048 arcs)
        src[:4000] = 5
        y = synth.uniform_labels(n, k, seed=3, device=dev)
        exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), None if w is None else w.cpu().numpy(),
                                  y.cpu().numpy(), n, k)
        g = DeviceGraph.from_edges(src, dst, w, n, pull=True, keep_coo=True)
        g.prepare_hot(k, enable=True)
        assert g.n_heavy > 0 and g.n_hot >= 16384, (g.n_heavy, g.n_hot)
        emb = Embedder(n, k)
        emb.project(y, g=g)
        check(emb.pull(g), exp, f"pull blocks+heavy weighted={weighted}")
        check(emb.embed(g, y, variant="push"), exp, f"push weighted={weighted}")
        pipe = HostPipeline(g, k, chunks=3)
        h_z = pinned_like((n, k))
        pipe.run(y.cpu().pin_memory(), h_z, emb)
        check(h_z.numpy(), exp, f"host pipeline packed weighted={weighted}")
        torch.cuda.synchronize()
    # wide reducer (K > 255): light rows + one heavy row
    k = 300
    src, dst, w = synth.rmat_edges(scale, s, seed=4, weighted=True, device=dev)
    src[:3000] = 9
    y = synth.uniform_labels(n, k, seed=4, device=dev)
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), w.cpu().numpy(), y.cpu().numpy(), n, k)
    g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
    emb = Embedder(n, k)
    assert emb.reducer_for(g) == "wide"
    check(emb.embed(g, y, variant="pull"), exp, "wide pull")
    torch.cuda.synchronize()
    print("sanitize_run: done")


if __name__ == "__main__":
    main()
