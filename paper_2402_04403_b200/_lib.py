"""ctypes binding of libgee_b200.so (the C ABI declared in include/gee_b200.h).

The library is the product path.  If it is missing, importing this module
raises: there is no CPU fallback.
"""

import ctypes
import os

from .errors import GeeError, ValidationError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libgee_b200.so")

GEE_OK = 0
GEE_ERR_INVALID = 1
GEE_ERR_CUDA = 2
GEE_ERR_RANGE = 3

GEE_ZERO_Z = 1
GEE_SOURCE_ONLY = 2
GEE_PRECOMBINE = 4

c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
c_size = ctypes.c_size_t
c_dbl = ctypes.c_double
vp = ctypes.c_void_p
P_dbl = ctypes.POINTER(ctypes.c_double)
P_i32 = ctypes.POINTER(ctypes.c_int32)

# name -> (restype, argtypes); every symbol include/gee_b200.h and
# include/gee_synth.h declare.
SIGNATURES = {
    "gee_version": (c_int, []),
    "gee_last_error": (ctypes.c_char_p, []),
    "gee_label_bytes": (c_int, [c_i32]),
    "gee_label_table_bytes": (c_size, [c_i64, c_i64, c_i32]),
    "gee_projection_work_bytes": (c_size, [c_i32]),
    "gee_build_projection": (c_int, [vp, c_i64, c_i32, vp, vp, vp, vp, vp, c_i64, vp, vp]),
    "gee_build_projection_hotc": (c_int, [vp, c_i64, c_i32, vp, vp, vp, vp, vp, vp, vp, c_i64, vp, vp]),
    "gee_build_projection_sharded": (c_int, [vp, c_i64, c_i32, vp, vp, vp, vp, vp, c_i64, c_i64, c_i64, vp, vp]),
    "gee_projection_inv": (c_int, [vp, c_i32, vp, vp, vp]),
    "gee_embed_coo": (c_int, [vp, vp, vp, c_i64, vp, c_i64, vp, c_i64, c_i32, vp, c_u32, vp]),
    "gee_build_csr": (c_int, [vp, vp, vp, c_i64, c_i64, c_i32, c_i32, vp, vp, vp, vp]),
    "gee_build_sym_csr": (c_int, [vp, vp, vp, c_i64, c_i64, vp, vp, vp, vp]),
    "gee_sym_offsets": (c_int, [vp, vp, c_i64, c_i64, vp, vp]),
    "gee_build_sym_csr_rows": (c_int, [vp, vp, vp, c_i64, c_i64, c_i64, c_i64, vp, vp, vp, vp, vp]),
    "gee_csr_rows": (c_int, [vp, c_i64, c_i64, vp, vp]),
    "gee_graph_stats": (c_int, [vp, vp, c_i64, c_i64, P_dbl, P_dbl, P_dbl, P_i32, vp]),
    "gee_hot_plan": (c_int, [vp, c_i64, c_i64, c_i64, vp, vp, ctypes.POINTER(c_i64), vp]),
    "gee_hot_encode": (c_int, [vp, c_i64, vp, c_i64, vp]),
    "gee_gather_labels": (c_int, [vp, c_i64, vp, c_i64, c_i32, vp, vp]),
    "gee_gather_labels_head": (c_int, [vp, c_i64, vp, c_i64, c_i32, c_i64, vp, vp]),
    "gee_widen_offsets": (c_int, [vp, c_i64, vp, vp]),
    "gee_zc_blocks": (c_i64, [c_i64]),
    "gee_z_compact": (c_int, [vp, c_i64, c_i32, vp, vp, vp, vp]),
    "gee_unpack_scratch_bytes": (c_size, [c_i64]),
    "gee_pack_targets": (c_int, [vp, c_i64, vp, vp, c_i64, c_i32, vp, vp, ctypes.POINTER(c_i64), vp, vp,
                                 ctypes.POINTER(c_i64), vp]),
    "gee_unpack_targets": (c_int, [vp, vp, c_i64, vp, c_i64, vp, c_i32, vp, c_i32, vp, vp, vp, c_size, vp]),
    "gee_reduce_wide": (c_int, [vp, c_i64, vp, vp, vp, c_i32, c_i32, vp, vp, c_i64, vp, vp]),
    "gee_reduce_heavy_plan": (c_int, [vp, c_i64, c_i64, vp, ctypes.POINTER(c_i64), vp]),
    "gee_pad_offsets": (c_int, [vp, c_i64, c_i64, vp, vp, vp]),
    "gee_pad_rows": (c_int, [vp, vp, c_i64, vp, vp, c_i32, vp, vp, vp]),
    "gee_sort_rows": (c_int, [vp, c_i64, vp, vp, vp]),
    "gee_reduce_blocks_pad8": (c_int, [vp, c_i64, vp, vp, c_i32, vp, c_i32, c_i64, vp, vp]),
    "gee_reduce_blocks_light": (c_int, [vp, c_i64, vp, vp, c_i32, vp, c_i32, vp, vp]),
    "gee_reduce_blocks_short": (c_int, [vp, c_i64, vp, vp, c_i32, vp, c_i32, vp, c_i32, vp, vp]),
    "gee_reduce_heavy": (c_int, [vp, vp, c_i64, c_i32, vp, c_i32, vp, vp, vp, vp, c_i64, vp, c_i64, vp, vp, vp, vp]),
    "gee_block_scale_exp": (c_int, [c_dbl, c_dbl, c_dbl, P_i32, P_dbl]),
    "gee_tile_bounds": (c_int, [vp, vp, c_i64, vp, vp, c_i32, vp, vp]),
    "gee_span_copy": (c_int, [c_i64, vp, vp, vp, vp, vp, vp, c_i32, vp, vp, vp]),
    "gee_gather_tiles": (c_int, [vp, vp, c_i32, c_i64, vp, vp, c_i64, c_i64, c_i32, vp, vp]),
    "gee_gather_scatter": (c_int, [vp, c_i64, c_i64, c_i64, vp, vp, c_i32, vp, vp]),
    "gee_synth_word": (c_u64, [c_u64, c_u64, c_u64]),
    "gee_synth_rmat": (c_int, [vp, vp, vp, c_i64, c_i64, c_i32, c_dbl, c_dbl, c_dbl, c_u64, c_i32, vp]),
    "gee_synth_er": (c_int, [vp, vp, vp, c_i64, c_i64, c_i64, c_u64, vp]),
    "gee_synth_uniform_labels": (c_int, [vp, c_i64, c_i32, c_u64, vp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the GEE edge pass has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class CudaError(GeeError):
    """A CUDA runtime or launch failure inside libgee_b200.so."""


def check(rc, what=""):
    """Raise the package error matching a C status code."""
    if rc == GEE_OK:
        return
    msg = lib.gee_last_error().decode("utf-8", "replace")
    if what:
        msg = f"{what}: {msg}"
    if rc in (GEE_ERR_INVALID, GEE_ERR_RANGE):
        raise ValidationError(msg)
    raise CudaError(msg)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
