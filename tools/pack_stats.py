"""Sizes of candidate target codes for the streamed e2e path on C4 (dev tool).

For the prepared C4 targets (slot-sorted rows, padded to 8) this sums, over
the real arcs only:
  * byte-width group deltas (gee_pack_targets today: 1 ctl byte per group);
  * bit-width group deltas (a group of 8 stores each delta in b bits, b the
    widest delta of the group; 1 ctl byte);
  * the same with the row's first value coded against the previous row's
    first value (zigzag);
  * a per-row Elias-Fano bound (2 + ceil(log2(range / d)) bits per arc).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph  # noqa: E402


def main():
    src, dst, w, y, n, k, _ = synth.make_config(4)
    g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
    del src, dst, w
    torch.cuda.empty_cache()
    g.prepare_hot(k)
    t, off = g.targets, g.offsets
    arcs = t.numel()
    sentinel = g.n_hot + n
    starts = torch.zeros(arcs + 1, dtype=torch.bool, device=t.device)
    nz = off[1:] > off[:-1]
    starts[off[:-1][nz]] = True
    out = {"arcs_padded": arcs, "rows_nonempty": int(nz.sum())}
    byte_b = bit_b = bit_first_b = 0
    real = 0
    step = 1 << 27
    prev_first = 0
    for a in range(0, arcs, step):
        b = min(arcs, a + step)
        x = t[a:b].long()
        prev = torch.empty_like(x)
        prev[1:] = x[:-1]
        prev[0] = t[a - 1].long() if a else 0
        st = starts[a:b]
        d = torch.where(st, x, x - prev)
        pad = x == sentinel
        d = torch.where(pad, torch.zeros_like(d), d)
        realm = ~pad
        real += int(realm.sum())
        nbytes = torch.where(d < (1 << 8), 1, torch.where(d < (1 << 16), 2, torch.where(d < (1 << 24), 3, 4)))
        nbits = (torch.floor(torch.log2(d.double().clamp(min=1))) + 1).long()
        gcount = realm.view(-1, 8).sum(1)
        gbyte = torch.where(realm, nbytes, 0).view(-1, 8).amax(1)
        gbit = torch.where(realm, nbits, 0).view(-1, 8).amax(1)
        byte_b += int((gbyte * gcount).sum()) + gbyte.numel()  # + ctl byte per group
        bit_b += int((gbit * gcount).sum() + 7) // 8 + gbit.numel()
        # first value of a row against the previous row's first value (zigzag)
        firsts = x[st]
        pf = torch.empty_like(firsts)
        if firsts.numel():
            pf[1:] = firsts[:-1]
            pf[0] = prev_first
            prev_first = int(firsts[-1])
        zz = firsts - pf
        zz = torch.where(zz >= 0, 2 * zz, -2 * zz - 1)
        d2 = d.clone()
        d2[st] = zz
        nbits2 = (torch.floor(torch.log2(d2.double().clamp(min=1))) + 1).long()
        gbit2 = torch.where(realm, nbits2, 0).view(-1, 8).amax(1)
        bit_first_b += int((gbit2 * gcount).sum() + 7) // 8 + gbit2.numel()
    out["real_arcs"] = real
    out["byte_width_GB"] = byte_b / 1e9
    out["bit_width_GB"] = bit_b / 1e9
    out["bit_width_first_vs_prev_GB"] = bit_first_b / 1e9
    # Elias-Fano bound per row: d * (2 + ceil(log2(max(1, range / d))))
    deg_real = torch.zeros(n, dtype=torch.int64, device=t.device)
    # real degree per row: padded length minus pads (pads are at the row end)
    plen = off[1:] - off[:-1]
    last = t[(off[1:] - 1).clamp(min=0)].long()
    # count pads per row exactly: pads are the sentinel arcs at the end, < 8
    npads = torch.zeros(n, dtype=torch.int64, device=t.device)
    for j in range(1, 8):
        idx = (off[1:] - j).clamp(min=0)
        ispad = (t[idx].long() == sentinel) & (plen >= j)
        npads += ispad.long()
    deg_real = plen - npads
    nzr = deg_real > 0
    first = t[off[:-1].clamp(max=arcs - 1)].long()
    lastr = t[(off[:-1] + deg_real - 1).clamp(min=0, max=arcs - 1)].long()
    rng = (lastr - first + 1).clamp(min=1)
    dd = deg_real.clamp(min=1)
    lowb = torch.clamp(torch.ceil(torch.log2((rng.double() / dd.double()).clamp(min=1))), min=0)
    ef_bits = torch.where(nzr, dd * (2 + lowb.long()) + 32, 0)  # + 32 bits for the row's first value
    out["elias_fano_GB"] = float(ef_bits.sum()) / 8e9
    out["current_bytes_per_arc"] = byte_b / real
    out["bit_width_bytes_per_arc"] = bit_b / real
    out["ef_bytes_per_arc"] = float(ef_bits.sum()) / 8 / real
    print(json.dumps(out), flush=True)
    del deg_real, last


if __name__ == "__main__":
    main()
