"""Compressible-memory probe on C4 (dev tool).

B200 supports generic data compression for allocations made with
cuMemCreate(compressionType = CU_MEM_ALLOCATION_COMP_GENERIC): the memory
system stores compressible sectors (zeros, small values) in fewer DRAM
bytes.  Z is mostly zeros (74M of C4's 134M rows are empty, a nonempty row
holds a few of its 50 classes), and the class stream holds bytes < 64.
This times the pull with Z / the class stream / the CSR arrays placed in
compressible allocations against plain ones, and checks Z bit for bit."""
import json
import sys

import torch
from cuda.bindings import driver as drv

sys.path.insert(0, ".")
from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402


def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) == 2 else r


class CompBuf:
    def __init__(self, nbytes, dtype, shape, comp=True):
        dev = torch.cuda.current_device()
        prop = drv.CUmemAllocationProp()
        prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        if comp:
            prop.allocFlags.compressionType = drv.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_GENERIC
        gran = ok(drv.cuMemGetAllocationGranularity(
            prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
        size = (nbytes + gran - 1) // gran * gran
        self.handle = ok(drv.cuMemCreate(size, prop, 0))
        self.ptr = ok(drv.cuMemAddressReserve(size, 0, 0, 0))
        ok(drv.cuMemMap(self.ptr, size, 0, self.handle, 0))
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        ok(drv.cuMemSetAccess(self.ptr, size, [acc], 1))
        got = drv.CUmemAllocationProp()
        got = ok(drv.cuMemGetAllocationPropertiesFromHandle(self.handle))
        self.compressed = int(got.allocFlags.compressionType) == 1
        typestr = {torch.float32: "<f4", torch.uint8: "|u1", torch.int32: "<i4", torch.int64: "<i8"}[dtype]
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(self.ptr), False), "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device="cuda")


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.cuda.current_device()
    sup = ok(drv.cuDeviceGetAttribute(
        drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, dev))
    out = {"generic_compression_supported": int(sup)}
    print(json.dumps(out), flush=True)
    src, dst, w, y, n, k, directed = synth.make_config(4)
    g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
    del src, dst, w
    torch.cuda.empty_cache()
    g.prepare_hot(k)
    emb = Embedder(n, k)
    emb.project(y, g=g)
    z_ref = emb.pull(g)
    step = lambda z: (emb.project(y, validate=False, g=g), emb.pull(g, z))  # noqa: E731
    out["plain_ms"] = timeit(lambda: step(z_ref))
    print(json.dumps(out), flush=True)
    # control: Z in a plain cuMemCreate allocation (same mapping path, no compression)
    zp = CompBuf(n * k * 4, torch.float32, (n, k), comp=False)
    out["z_vmm_plain_ms"] = timeit(lambda: step(zp.tensor))
    out["z_vmm_plain_same"] = bool(torch.equal(zp.tensor, z_ref))
    del zp
    # Z compressible
    zb = CompBuf(n * k * 4, torch.float32, (n, k))
    out["z_alloc_compressed"] = zb.compressed
    out["z_comp_ms"] = timeit(lambda: step(zb.tensor))
    out["z_same"] = bool(torch.equal(zb.tensor, z_ref))
    print(json.dumps(out), flush=True)
    # class stream compressible too
    cb = CompBuf(emb.cls.numel(), torch.uint8, (emb.cls.numel(),))
    cls_plain = emb.cls
    emb.cls = cb.tensor
    out["z_cls_comp_ms"] = timeit(lambda: step(zb.tensor))
    out["z_cls_same"] = bool(torch.equal(zb.tensor, z_ref))
    print(json.dumps(out), flush=True)
    emb.cls = cls_plain
    del cb
    # CSR targets / weights compressible (copies)
    tb = CompBuf(g.targets.numel() * 4, torch.int32, (g.targets.numel(),))
    tb.tensor.copy_(g.targets)
    t_plain = g.targets
    g.targets = tb.tensor
    out["z_tgt_comp_ms"] = timeit(lambda: step(zb.tensor))
    out["z_tgt_same"] = bool(torch.equal(zb.tensor, z_ref))
    g.targets = t_plain
    del tb
    print(json.dumps(out), flush=True)
    if g.weights is not None:
        wb = CompBuf(g.weights.numel() * 4, torch.float32, (g.weights.numel(),))
        wb.tensor.copy_(g.weights)
        w_plain = g.weights
        g.weights = wb.tensor
        out["z_w_comp_ms"] = timeit(lambda: step(zb.tensor))
        out["z_w_same"] = bool(torch.equal(zb.tensor, z_ref))
        g.weights = w_plain
        del wb
    out["plain_again_ms"] = timeit(lambda: step(z_ref))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
