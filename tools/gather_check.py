"""gee_gather_labels under every GEE_GATHER_MODE equals torch's gather (dev tool)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, torch
sys.path.insert(0, "@ROOT@")
from paper_2402_04403_b200 import _lib
g = torch.Generator(device="cuda").manual_seed(3)
n_hot, n = 300_000, 2_000_000
for k, arcs in ((50, 0), (50, 5), (50, 511), (50, 512 * 148 * 32 + 77), (50, 10_000_003), (5, 3_000_001),
                (20, 3_000_001), (63, 3_000_001), (64, 3_000_001), (200, 3_000_001)):
    table = torch.randint(0, k + 1, (n_hot + n + 1,), dtype=torch.uint8, device="cuda", generator=g)
    # skewed slots: half in the first 4096, a quarter in the hot tier, the rest anywhere
    u = torch.rand(arcs, device="cuda", generator=g)
    t = torch.where(u < 0.5, (u * 8192).long(), torch.where(u < 0.75, (u * n_hot).long() % n_hot,
                    torch.randint(0, n_hot + n + 1, (arcs,), device="cuda", generator=g)))
    t = t.int()
    cls = torch.full((arcs + 16,), 255, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib.gee_gather_labels(_lib.ptr(t), arcs, _lib.ptr(table), n_hot, k, _lib.ptr(cls),
                                          _lib.stream_handle()), "gather")
    torch.cuda.synchronize()
    assert torch.equal(cls[:arcs], table[t.long()]), arcs
    assert bool((cls[arcs:] == 255).all()), arcs
print("ok")
""".replace("@ROOT@", ROOT)

for env in ({}, {"GEE_GATHER_SMEM_HOT": "0"}, {"GEE_GATHER_SMEM_HOT": "40000"}, {"GEE_GATHER_SMEM_HOT": "131072"}):
    r = subprocess.run([sys.executable, "-c", CHILD], env={**os.environ, **env}, capture_output=True, text=True)
    print(env, r.stdout.strip(), r.stderr.strip()[-300:])
