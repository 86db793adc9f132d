"""ctypes binding of libfpx_sm100.so (include/fpx.h).

The library is built in-tree by `paper_2501_12349_b200.build` (also run by
`__graft_entry__.build()`).  There is no fallback: if the library or a CUDA
device is missing, every entry point raises `FpxNativeError`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPX_LIB") or os.path.join(HERE, "lib", "libfpx_sm100.so")
ABI_VERSION = 7

INTERIOR, BORDER, NOT_FOUND = 0, 1, 2
STAT_NAMES = ["points", "box_tests", "newton", "iters", "rest_points", "r1_warp_evals",
              "r1_w2_evals", "evals", "newton_r1", "iters_r1", "evals_r1", "r1_items",
              "rest_warp_evals", "rest_w2_evals", "rest_lane_evals", "redo", "r1_lane_evals"]
STATS_LEN = len(STAT_NAMES)
FREC = 32            # FPX_FREC: doubles per element filter record
FROW = 20            # FPX_FROW: floats per element pre-test row

P = C.c_void_p


class FpxNativeError(RuntimeError):
    """The CUDA library is missing, or a native call failed."""


class MeshT(C.Structure):
    """Mirror of `fpx_mesh_t` (include/fpx.h)."""

    _fields_ = [
        ("d", C.c_int32), ("dr", C.c_int32), ("N", C.c_int32), ("M", C.c_int32),
        ("E", C.c_int64),
        ("basis", P), ("nodes", P), ("aabb", P), ("obb_c", P), ("obb_inv", P), ("obb_ok", P),
        ("frame", P), ("grid", P),
        ("ncell", C.c_int32), ("max_list", C.c_int32),
        ("offsets", P), ("elems", P),
        ("max_iters", C.c_int32),
        ("tol", C.c_double), ("grow", C.c_double), ("keep", C.c_double),
        ("accept", C.c_double), ("shrink", C.c_double), ("alpha0", C.c_double),
        ("eps_d_abs", C.c_double), ("eps_d_rel", C.c_double),
        ("frec", P), ("nodes_pad", P),
        ("fbox", P),
    ]


_lib = None


def lib():
    """Load and type the native library (raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FpxNativeError(
            f"{LIB_PATH} not built; run `python -m paper_2501_12349_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    i32, i64, f64, sz = C.c_int, C.c_int64, C.c_double, C.c_size_t
    sig = {
        "fpx_abi_version": ([], i32),
        "fpx_last_error": ([], C.c_char_p),
        "fpx_supported": ([i32, i32, i32], i32),
        "fpx_launch_count": ([], i64),
        "fpx_profile_round1": ([P, P], i32),
        "fpx_probe_fp64": ([P, P], i32),
        "fpx_setup_bounds": ([i32, i32, i32, i32, i64, P, P, f64, P, P, P, P, P, P, P, P], i32),
        "fpx_filter_records": ([i32, i64, P, P, P, P, P, P, P, P], i32),
        "fpx_pad_nodes": ([i32, i32, i32, i64, P, P, P], i32),
        "fpx_set_round1_event": ([P], i32),
        "fpx_rest_patch_host": ([i32, i32, i64, i64, i64, P, C.c_size_t, C.POINTER(MeshT), P, P,
                                 P, P, P, P, P, P, P, P, P], i32),
        "fpx_set_upload_events": ([i32, P], i32),
        "fpx_set_round1_events": ([i32, P], i32),
        "fpx_set_find_hint": ([P], i32),
        "fpx_particles_advance": ([i32, i64, P, P, P, P, P, f64, f64, i32, P, i32, P], i32),
        "fpx_bound_function": ([i32, i32, i32, i64, P, P, P, P, P], i32),
        "fpx_hash_workspace_bytes": ([i32, i64, i32], sz),
        "fpx_hash_build": ([i32, i64, P, P, P, P, i32, P, P, P, i64, P, P, P, sz, P], i32),
        "fpx_cell_of": ([C.POINTER(MeshT), i64, P, P, P], i32),
        "fpx_find_workspace_bytes": ([C.POINTER(MeshT), i64, i64], sz),
        "fpx_find": ([C.POINTER(MeshT), i64, P, P, P, P, P, P, P, i32, P, P, i64, P, sz, P], i32),
        "fpx_eval_workspace_bytes": ([i64, i64], sz),
        "fpx_findpts_eval": ([i32, i32, P, i32, i64, P, i64, P, P, P, P, P, sz, P], i32),
        "fpx_invert_pairs": ([C.POINTER(MeshT), i64, P, P, P, P, P, P, P, P], i32),
        "fpx_forward_map": ([C.POINTER(MeshT), i64, P, P, P, P, P, P], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.fpx_abi_version() != ABI_VERSION:
        raise FpxNativeError(f"ABI mismatch: library {L.fpx_abi_version()} != {ABI_VERSION}")
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/fpx.h (checked by the CPU test suite)."""
    return ["fpx_abi_version", "fpx_last_error", "fpx_launch_count", "fpx_profile_round1",
            "fpx_probe_fp64", "fpx_supported", "fpx_setup_bounds", "fpx_filter_records", "fpx_pad_nodes",
            "fpx_particles_advance", "fpx_set_round1_event", "fpx_rest_patch_host", "fpx_set_upload_events",
            "fpx_set_round1_events",
            "fpx_set_find_hint",
            "fpx_bound_function", "fpx_hash_workspace_bytes", "fpx_hash_build", "fpx_cell_of",
            "fpx_find_workspace_bytes", "fpx_find", "fpx_eval_workspace_bytes",
            "fpx_findpts_eval", "fpx_invert_pairs", "fpx_forward_map"]


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().fpx_last_error().decode(errors="replace")
        raise FpxNativeError(f"{what} failed ({rc}): {msg}")


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise FpxNativeError("no CUDA device: the fpx hot path runs only on the GPU "
                             "(no CPU fallback)")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def stream_handle(stream: torch.cuda.Stream | None = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def pack_basis(bc) -> np.ndarray:
    """Packed per-order constants in the FPX_BASIS_* layout."""
    return np.concatenate([bc.nodes, bc.scale, bc.proj0, bc.proj1, bc.eta,
                           np.asarray(bc.lo).reshape(-1), np.asarray(bc.hi).reshape(-1)])
