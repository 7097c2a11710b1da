"""ctypes binding of the C ABI in ``include/skr.h`` (libskr.so).

The product path has no CPU fallback: if the extension is missing or no CUDA
device is present, every entry point raises ``SkrExtensionError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from ctypes import POINTER, c_double, c_int32, c_int64, c_size_t, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
# SKR_LIB_PATH: load another build (A/B measurements of older revisions)
LIB_PATH = os.environ.get("SKR_LIB_PATH") or os.path.join(PKG, "libskr.so")

EXPORTS = (
    "skr_version", "skr_status_string", "skr_device_info", "skr_spmv", "skr_residual",
    "skr_stencil_bytes", "skr_stencil_build", "skr_assemble_fd",
    "skr_grf_workspace_bytes", "skr_grf_sample", "skr_philox_normals", "skr_philox_uniforms",
    "skr_gcrodr_workspace_bytes", "skr_gcrodr_solve", "skr_gcrodr_recycle_view",
    "skr_gcrodr_profile", "skr_gcrodr_solve_chains", "skr_gcrodr_diagnostics",
    "skr_sort_workspace_bytes", "skr_sort_binary_check", "skr_sort_dist2", "skr_sort_chain",
    "skr_greedy_sort", "skr_dense_hr_first", "skr_dense_hr_next",
    "skr_precond_bytes", "skr_precond_build", "skr_precond_apply",
    "skr_sort_pca_workspace_bytes", "skr_sort_pca_keys",
)


class SkrExtensionError(RuntimeError):
    """The CUDA extension is missing or failed; there is no fallback path."""


class SkrCsr(ctypes.Structure):
    _fields_ = [("n", c_int32), ("nnz", c_int32), ("row_ptr", c_void_p),
                ("col_idx", c_void_p), ("values", c_void_p), ("diag", c_void_p),
                ("stencil", c_void_p), ("sx", c_int32), ("sxy", c_int32),
                ("precond", c_void_p), ("precond_kind", c_int32)]


class SkrSystem(ctypes.Structure):
    _fields_ = [("A", SkrCsr), ("b", c_void_p), ("x", c_void_p)]


class SkrConfig(ctypes.Structure):
    _fields_ = [("m", c_int32), ("k", c_int32), ("max_iter", c_int32),
                ("grid_ctas", c_int32), ("tol", c_double), ("flags", c_int32)]


COLLECT_DIAGNOSTICS = 1


class SkrReport(ctypes.Structure):
    _fields_ = [("iterations", c_int32), ("converged", c_int32), ("k_out", c_int32),
                ("hist_len", c_int32), ("n_checks", c_int32), ("deflated_steps", c_int32),
                ("warn_bits", c_int32), ("status_bits", c_int32), ("zero_rhs", c_int32),
                ("gmres_fallback", c_int32), ("cycles", c_int32), ("v0_projections", c_int32),
                ("true_relative_residual", c_double), ("rnorm", c_double),
                ("abs_tol", c_double), ("bnorm", c_double), ("device_ms", c_double),
                ("spmv_ortho_bytes", c_double), ("cycle_kernel_ms", c_double),
                ("dense_kernel_ms", c_double), ("launches", c_int32),
                ("arnoldi_steps", c_int32)]


PC_KINDS = {"sor": 1, "ilu0": 2, "icc0": 3, "bjacobi": 4}

WARN_SINGULAR_H = 1
WARN_SINGULAR_CROSS = 2
WARN_RANK_DROP = 4
WARN_REFRESH_RANK = 8
WARN_JACOBI_SVD = 16

_lock = threading.Lock()
_lib = None


def _declare(L):
    P = c_void_p
    sig = {
        "skr_version": ([], c_int32),
        "skr_status_string": ([c_int32], ctypes.c_char_p),
        "skr_device_info": ([POINTER(c_int32), POINTER(c_int64)], c_int32),
        "skr_spmv": ([POINTER(SkrCsr), P, P, c_int32, P], c_int32),
        "skr_stencil_bytes": ([c_int32, c_int32, c_int32], ctypes.c_size_t),
        "skr_stencil_build": ([POINTER(SkrCsr), c_int32, c_int32, P, ctypes.c_size_t, P], c_int32),
        "skr_assemble_fd": ([c_int32, c_int32, c_int32, P, c_double, P, P, P, ctypes.c_size_t, P],
                            c_int32),
        "skr_residual": ([POINTER(SkrCsr), P, P, P, c_int32, P], c_int32),
        "skr_grf_workspace_bytes": ([c_int32, c_int32], c_size_t),
        "skr_grf_sample": ([c_int32, c_int32, c_int32, c_double, c_double, c_double, P,
                            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, P, P, P, c_size_t,
                            P], c_int32),
        "skr_philox_normals": ([c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                ctypes.c_uint32, c_double, P, P], c_int32),
        "skr_philox_uniforms": ([c_int32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                 ctypes.c_uint32, P, P], c_int32),
        "skr_gcrodr_workspace_bytes": ([c_int32, c_int32, c_int32, c_int32], c_size_t),
        "skr_gcrodr_solve": ([POINTER(SkrCsr), P, P, P, POINTER(SkrConfig), P, c_int32, c_int32,
                              P, c_size_t, POINTER(SkrReport), P, c_int32, P, c_int32, P],
                             c_int32),
        "skr_gcrodr_recycle_view": ([P, c_size_t, c_int32, c_int32, c_int32, POINTER(c_void_p),
                                     POINTER(c_void_p), POINTER(c_int32), POINTER(c_int32)],
                                    c_int32),
        "skr_gcrodr_profile": ([P, c_size_t, c_int32, c_int32, c_int32, P], c_int32),
        "skr_gcrodr_diagnostics": ([P, c_size_t, c_int32, c_int32, c_int32, c_int32, P, c_int32],
                                   c_int32),
        "skr_gcrodr_solve_chains": ([POINTER(SkrSystem), P, c_int32, POINTER(SkrConfig), P,
                                     c_size_t, P, P, P, POINTER(SkrReport)], c_int32),
        "skr_sort_workspace_bytes": ([c_int32, c_int64], c_size_t),
        "skr_sort_binary_check": ([P, c_int32, c_int64, P, POINTER(c_int32), P, c_size_t, P],
                                  c_int32),
        "skr_sort_dist2": ([P, c_int32, c_int64, c_int32, c_int32, c_int32, c_double, c_double,
                            P, P, c_size_t, P], c_int32),
        "skr_sort_chain": ([P, P, c_int32, c_int64, c_int32, P, P, P], c_int32),
        "skr_greedy_sort": ([P, c_int32, c_int64, P, P, c_size_t, P], c_int32),
        "skr_dense_hr_first": ([P, c_int32, c_int32, c_int32, P, c_int32, POINTER(c_int32), P],
                               c_int32),
        "skr_dense_hr_next": ([P, c_int32, P, c_int32, c_int32, c_int32, P, c_int32,
                               POINTER(c_int32), P], c_int32),
        "skr_sort_pca_workspace_bytes": ([c_int32], c_size_t),
        "skr_sort_pca_keys": ([P, P, c_int32, c_int64, P, P, c_size_t, P], c_int32),
        "skr_precond_bytes": ([c_int32, c_int32, c_int32, c_int32], c_size_t),
        "skr_precond_build": ([POINTER(SkrCsr), c_int32, c_double, c_int32, P, c_size_t,
                               POINTER(c_int32), POINTER(c_double), P], c_int32),
        "skr_precond_apply": ([P, P, P, c_int32, c_int64, c_int64, P], c_int32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res


def load(build_if_missing: bool = True):
    """Load (and if needed build) libskr.so. Raises SkrExtensionError."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH) and build_if_missing:
            try:
                from . import _build
                _build.build_cuda(verbose=False)
            except Exception as e:  # pragma: no cover - depends on toolchain
                raise SkrExtensionError(f"libskr.so missing and build failed: {e}") from e
        if not os.path.exists(LIB_PATH):
            raise SkrExtensionError(f"libskr.so not found at {LIB_PATH}")
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as e:
            raise SkrExtensionError(f"cannot load {LIB_PATH}: {e}") from e
        _declare(L)
        _lib = L
        return L


def check(status: int, what: str):
    if status != 0:
        msg = load().skr_status_string(status).decode()
        raise SkrExtensionError(f"{what} failed: {msg} (status {status})")


def require_cuda():
    """Fail loudly unless a CUDA device is usable (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise SkrExtensionError("no CUDA device: the SKR hot path runs only on the GPU")
    load()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
