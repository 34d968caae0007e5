"""ctypes binding of libhsseig_b200.so (the C ABI declared in include/hsseig_b200.h).

There is no CPU fallback: importing the compute entry points without the built
library, or calling them without a CUDA device, raises immediately.
"""
import ctypes
import os

import torch

from . import build as _build

_LIB = None

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

HSSEIG_OK = 0
HSSEIG_ERR_ARG = 1
HSSEIG_ERR_BRACKET = 2
HSSEIG_ERR_RADICAND = 3
HSSEIG_ERR_CUDA = 4


class Gen(ctypes.Structure):
    """hsseig_gen"""
    _fields_ = [("d", c_vp), ("dnext", c_vp), ("gamma", c_vp), ("mu", c_vp), ("zhat", c_vp),
                ("v", c_vp), ("k", c_i64)]


class Tree(ctypes.Structure):
    """hsseig_tree"""
    _fields_ = [("k", c_i32), ("n_leaves", c_i32), ("depth", c_i32), ("n_nodes", c_i32),
                ("w", c_i32), ("ws", c_i32), ("pmax", c_i32), ("mmax", c_i32),
                ("lo", c_vp), ("hi", c_vp), ("left", c_vp), ("right", c_vp),
                ("level_nodes", c_vp), ("level_off", c_vp), ("level_off_h", c_i32 * 33),
                ("root", c_i32),
                ("rU", c_vp), ("rV", c_vp), ("rsel", c_vp), ("csel", c_vp), ("rloc", c_vp),
                ("cloc", c_vp), ("flags", c_vp),
                ("U", c_vp), ("V", c_vp), ("Vt", c_vp), ("B", c_vp), ("D", c_vp), ("rres", c_vp),
                ("cres", c_vp), ("dld", c_i32),
                ("M", c_vp), ("psel", c_vp), ("tsel", c_vp), ("ycomp", c_vp), ("zcomp", c_vp), ("rmax", c_i32),
                ("leaf_of", c_vp)]


# name -> (restype, argtypes)
_SIGS = {
    "hsseig_version": (ctypes.c_char_p, []),
    "hsseig_launch_count": (c_i64, []),
    "hsseig_last_error": (ctypes.c_char_p, []),
    "hsseig_status_init": (ctypes.c_int, [c_vp, c_i64, c_vp]),
    "hsseig_secular": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      c_vp, c_vp]),
    "hsseig_secular_part": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, c_i64, c_i64, c_vp, c_vp,
                                           c_vp, c_vp, c_vp, c_vp, c_vp]),
    "hsseig_loewner_part": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_i64,
                                           c_i64, c_vp, c_vp, c_vp]),
    "hsseig_normalizers_part": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                                               c_vp, c_vp]),
    "hsseig_cauchy_sample_part": (ctypes.c_int, [ctypes.POINTER(Gen), c_vp, c_vp, c_i64, c_i64,
                                                 c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "hsseig_cauchy_sample_part_peers": (ctypes.c_int, [ctypes.POINTER(Gen), c_vp, c_vp, c_i64,
                                                       c_i64, c_i64, c_i64, c_vp, c_vp, c_i32,
                                                       c_i64, c_vp, c_vp]),
    "hsseig_sample_peers_fits": (ctypes.c_int, [c_i64, c_i64, c_i64]),
    "hsseig_dnext": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "hsseig_loewner": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp,
                                      c_vp]),
    "hsseig_normalizers": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "hsseig_cauchy_block": (ctypes.c_int, [ctypes.POINTER(Gen), c_vp, c_i64, c_vp, c_i64, c_vp,
                                           c_i64, c_vp]),
    "hsseig_sample_work_doubles": (c_i64, [c_i64, c_i64]),
    "hsseig_cauchy_sample": (ctypes.c_int, [ctypes.POINTER(Gen), c_vp, c_vp, c_i64, c_i64, c_vp,
                                            c_vp, c_i64, c_vp, c_vp]),
    "hsseig_tree_bytes": (c_i64, [c_i32, c_i32, c_i32, c_i32]),
    "hsseig_tree_layout": (ctypes.c_int, [ctypes.POINTER(Tree), ctypes.POINTER(c_i32), c_i32,
                                          c_i32, c_vp, c_vp]),
    "hsseig_hss_build_rand": (ctypes.c_int, [ctypes.POINTER(Gen), c_vp, c_i64, c_vp, c_vp, c_i64,
                                             c_dbl, c_i32, ctypes.POINTER(Tree), c_vp, c_vp]),
    "hsseig_tree_clear": (ctypes.c_int, [ctypes.POINTER(Tree), c_vp]),
    "hsseig_interp_smem_bytes": (c_i64, [c_i32, c_i32]),
    "hsseig_interp_decomp": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i32, c_i32, c_i64, c_dbl, c_i32,
                                            c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "hsseig_hss_build_rand_levels": (ctypes.c_int, [ctypes.POINTER(Gen), c_vp, c_i64, c_vp, c_vp,
                                                    c_i64, c_dbl, c_i32, ctypes.POINTER(Tree), c_vp,
                                                    ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                    ctypes.c_int, c_vp]),
    "hsseig_srrsc_work_doubles": (c_i64, [ctypes.POINTER(Tree)]),
    "hsseig_hss_build_srrsc": (ctypes.c_int, [ctypes.POINTER(Gen), c_dbl, c_i32,
                                              ctypes.POINTER(Tree), c_vp, c_vp, c_vp]),
    "hsseig_hss_build_srrsc_levels": (ctypes.c_int, [ctypes.POINTER(Gen), c_dbl, c_i32,
                                                     ctypes.POINTER(Tree), c_vp, c_vp,
                                                     ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                     ctypes.c_int, c_vp]),
    "hsseig_matmul_work_doubles": (c_i64, [c_i64, ctypes.POINTER(Tree)]),
    "hsseig_hss_matmul_right": (ctypes.c_int, [c_vp, c_i64, c_i64, ctypes.POINTER(Tree), c_vp,
                                               c_i64, c_vp, c_vp]),
    "hsseig_hss_matmul_right_part": (ctypes.c_int, [c_vp, c_i64, c_i64, ctypes.POINTER(Tree), c_vp,
                                                    c_i64, c_vp, ctypes.c_int32, ctypes.c_int32, c_vp]),
    "hsseig_dense_update": (ctypes.c_int, [c_vp, c_i64, c_i64, ctypes.POINTER(Gen), c_vp, c_i64,
                                           c_vp]),
    "hsseig_dense_update_work_doubles": (c_i64, [c_i64, c_i64]),
    "hsseig_dense_update_ws": (ctypes.c_int, [c_vp, c_i64, c_i64, ctypes.POINTER(Gen), c_vp, c_i64,
                                              c_vp, c_i64, c_vp]),
    "hsseig_dense_update_halves_work_doubles": (c_i64, [c_i64, c_i64, c_i64]),
    "hsseig_dense_update_halves": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i64, ctypes.POINTER(Gen), c_vp,
                                                  c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "hsseig_wave_dense_halves": (ctypes.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                                c_vp, c_vp, c_vp, c_i64, ctypes.c_int32, c_vp]),
    "hsseig_set_normal_tables": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "hsseig_normals_work_bytes": (c_i64, [c_i64]),
    "hsseig_normals_fixup": (c_i64, [c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp]),
    "hsseig_pcg64_normals": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp,
                                            c_vp, c_i64, c_vp]),
    "hsseig_tql2_batched": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, ctypes.c_int, ctypes.c_int,
                                           c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp]),
    "hsseig_deflate": (c_i64, [c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                               c_vp, c_vp]),
    "hsseig_deflate_tol": (c_i64, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp, c_vp]),
    "hsseig_assemble_merge": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "hsseig_apply_rotations": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                              c_vp]),
    "hsseig_gather_columns": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64,
                                             c_vp, c_i64, c_vp]),
    "hsseig_gemm": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64,
                                   c_vp]),
    "hsseig_assemble_rows": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp,
                                            c_i64, c_vp]),
    "hsseig_wave_zrows": (ctypes.c_int, [c_vp] * 5 + [c_i64, c_vp, c_vp]),
    "hsseig_wave_deflate": (c_i64, [c_i64] + [c_vp] * 16),
    "hsseig_wave_compact": (c_i64, [c_i64] + [c_vp] * 10),
    "hsseig_wave_assemble": (ctypes.c_int, [c_vp] * 11 + [c_i64, c_vp]),
    "hsseig_wave_rotate": (ctypes.c_int, [c_vp] * 10 + [c_i64, c_i64, c_vp]),
    "hsseig_wave_secular": (ctypes.c_int, [c_vp] * 5 + [c_i64, c_i64] + [c_vp] * 7),
    "hsseig_wave_dnext": (ctypes.c_int, [c_vp] * 5 + [c_i64, c_vp, c_vp]),
    "hsseig_wave_loewner": (ctypes.c_int, [c_vp] * 8 + [c_i64, c_vp, c_vp, c_vp]),
    "hsseig_wave_normalizers": (ctypes.c_int, [c_vp] * 7 + [c_i64, c_vp, c_vp]),
    "hsseig_wave_dense_update": (ctypes.c_int, [c_vp] * 14 + [c_i64, c_vp]),
    "hsseig_wave_tile_shape": (ctypes.c_int, [c_vp, c_vp]),
    "hsseig_wave_order": (ctypes.c_int, [c_i64] + [c_vp] * 7),
    "hsseig_wave_desc": (ctypes.c_int, [c_i64] + [c_vp] * 6),
    "hsseig_wave_gather": (ctypes.c_int, [c_vp] * 15 + [c_i64, c_vp]),
    "hsseig_wave_gather_rows": (ctypes.c_int, [c_vp] * 15 + [c_i64, c_vp, c_vp]),
}

EXPORTS = tuple(_SIGS)


def lib_path():
    return _build.LIB


def load(build_if_missing=True):
    """Load (building first if stale and nvcc is present) the shared library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _build.LIB
    if build_if_missing:
        try:
            _build.build()
        except (OSError, FileNotFoundError):
            pass
    if not os.path.exists(path):
        raise RuntimeError(f"hsseig_b200: native library {path} is missing; run "
                           "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("hsseig_b200 requires a CUDA device (sm_100a); there is no CPU path")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def stream_ptr(stream=None):
    """cudaStream_t of `stream` (default: torch's current stream on the current device).  The
    raw-stream query skips torch.cuda.current_stream()'s Python wrapper (~16 us a call; 600
    calls per config-2 solve)."""
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    try:
        return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))
    except AttributeError:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def check(rc, what):
    if rc == HSSEIG_OK:
        return
    if rc == HSSEIG_ERR_ARG:
        detail = _LIB.hsseig_last_error().decode() if _LIB is not None else "invalid argument"
        raise ValueError(f"{what}: {detail}")
    raise RuntimeError(f"{what}: CUDA error (status {rc})")
