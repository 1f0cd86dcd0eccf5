"""ctypes binding of the C-ABI (include/w1mg_cuda.h).

Loads the in-tree paper_1810_00118_b200/lib/libw1mg_cuda.so and fails loudly
when it is missing: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
# W1MG_CUDA_SO: load another build of the library (engine A/B experiments)
CUDA_SO = os.environ.get("W1MG_CUDA_SO") or os.path.join(LIB_DIR, "libw1mg_cuda.so")
API_SO = os.path.join(LIB_DIR, "libw1mg.so")

W1MG_OK, W1MG_EINVAL, W1MG_ELOGIC, W1MG_ECUDA, W1MG_ENOMEM, W1MG_ENONFINITE = range(6)
P1, P2, PINF = 0, 1, 2
STEP_SAFE, STEP_PRACTICAL = 0, 1

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_long)
_ip = C.POINTER(C.c_int)


class CPReport(C.Structure):
    _fields_ = [("distance", C.c_double), ("dual_value", C.c_double), ("converged", C.c_int),
                ("iterations", C.c_long), ("fpr_final", C.c_double), ("seconds", C.c_double)]


class LevelStatsC(C.Structure):
    _fields_ = [("h", C.c_double), ("eps", C.c_double), ("iters", C.c_long),
                ("fpr_final", C.c_double), ("seconds", C.c_double)]


class MLParams(C.Structure):
    _fields_ = [("levels", C.c_int), ("pnorm", C.c_int), ("step_mode", C.c_int),
                ("rel_tol", C.c_double), ("eps", _dp), ("max_iters", C.c_long)]


class W1MGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lock = threading.Lock()
_lib = None


def build() -> None:
    import subprocess

    r = subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc")], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError("CUDA library build failed:\n" + r.stdout + r.stderr)


def lib():
    """The loaded libw1mg_cuda.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(CUDA_SO):
            raise ImportError(
                f"{CUDA_SO} is missing: run __graft_entry__.build() (make -C "
                "paper_1810_00118_b200/csrc). There is no CPU fallback.")
        L = C.CDLL(CUDA_SO)
        L.w1mg_last_error.restype = C.c_char_p
        L.w1mg_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.w1mg_ctx_destroy.argtypes = [C.c_void_p]
        L.w1mg_ctx_launch_count.argtypes = [C.c_void_p]
        L.w1mg_ctx_launch_count.restype = C.c_long
        L.w1mg_ctx_synchronize.argtypes = [C.c_void_p]
        L.w1mg_ctx_level_seconds.argtypes = [C.c_void_p, _dp, C.c_int]
        L.w1mg_ctx_stream.argtypes = [C.c_void_p]
        L.w1mg_ctx_stream.restype = C.c_void_p
        L.w1mg_cp_step_size.argtypes = [C.c_int, C.c_int]
        L.w1mg_cp_step_size.restype = C.c_double
        L.w1mg_pdhg_step_size.argtypes = [C.c_int]
        L.w1mg_pdhg_step_size.restype = C.c_double
        L.w1mg_make_schedule.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp]
        L.w1mg_source_check.argtypes = [C.c_int, _dp]
        L.w1mg_divergence.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.w1mg_adjoint.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.w1mg_primal_value.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_int, _dp]
        L.w1mg_inner_h_nodes.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.w1mg_inner_h_edges.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.w1mg_cp_run.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, C.c_int, C.c_double,
                                  C.c_double, C.c_double, C.c_long, _dp, _dp, _dp, _dp, C.c_long,
                                  C.POINTER(CPReport)]
        L.w1mg_cp_residual.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp,
                                       C.c_double, C.c_double, _dp]
        L.w1mg_ml_sources.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_int, _dp]
        L.w1mg_ml_cp_run.argtypes = [C.c_void_p, C.c_int, _dp, C.POINTER(MLParams), _dp, _dp, _dp,
                                     C.POINTER(LevelStatsC), _dp, C.c_long, C.POINTER(CPReport)]
        L.w1mg_ml_cp_batch.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp,
                                       C.POINTER(MLParams), _dp, _dp, _lp, _ip]
        L.w1mg_fp64_peak_probe.argtypes = [C.c_void_p, C.c_long, _dp]
        L.w1mg_ml_cp_batch_fields.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp,
                                              C.POINTER(MLParams), _dp, _dp, _lp, _ip, _dp, _dp,
                                              _dp, _dp]
        L.w1mg_ml_cp_batch_dev.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                           C.POINTER(MLParams), C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        L.w1mg_interpolate_scalar.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.w1mg_interpolate_flux.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp]
        L.w1mg_poisson_solve.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_int]
        L.w1mg_project_affine.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.w1mg_recover_potential.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.w1mg_pdhg_run.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                    C.c_int, C.c_double, C.c_double, C.c_double, C.c_long, _dp,
                                    _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_long,
                                    C.POINTER(CPReport)]
        L.w1mg_pdhg_residual.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                         _dp, C.c_double, C.c_double, _dp]
        L.w1mg_ml_pdhg_run.argtypes = [C.c_void_p, C.c_int, _dp, C.POINTER(MLParams), _dp, _dp,
                                       _dp, _dp, _dp, C.POINTER(LevelStatsC), _dp, C.c_long,
                                       C.POINTER(CPReport)]
        L.w1mg_slab_bounds.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.w1mg_nccl_unique_id.argtypes = [C.c_char_p]
        L.w1mg_slab_comm_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p,
                                            C.POINTER(C.c_void_p)]
        L.w1mg_slab_comm_destroy.argtypes = [C.c_void_p]
        L.w1mg_slab_comm_enable_peer.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.w1mg_set_slab_transport.argtypes = [C.c_int]
        L.w1mg_slab_cp_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp,
                                       _dp, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_long, _dp, _dp, _dp, _dp, C.c_long,
                                       C.POINTER(CPReport)]
        L.w1mg_ml_slab_cp_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _dp,
                                          C.POINTER(MLParams), _dp, _dp, _dp,
                                          C.POINTER(LevelStatsC), C.POINTER(CPReport)]
        L.w1mg_set_sweep_engine.argtypes = [C.c_int]
        L.w1mg_set_resident_engine.argtypes = [C.c_int]
        L.w1mg_set_tail_compaction.argtypes = [C.c_int]
        L.w1mg_set_pdhg_small.argtypes = [C.c_int]
        L.w1mg_set_option.argtypes = [C.c_char_p, C.c_long]
        _lib = L
        return L


def check(rc: int) -> None:
    if rc != W1MG_OK:
        msg = lib().w1mg_last_error().decode()
        if rc == W1MG_EINVAL:
            raise ValueError(msg)  # std::invalid_argument in the reference
        if rc == W1MG_ELOGIC:
            raise AssertionError(msg)  # std::logic_error("bad PNorm")
        if rc == W1MG_ENOMEM:
            raise MemoryError(msg)
        raise W1MGError(rc, msg)


def ptr(a):
    if a is None:
        return None
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise TypeError("expected a C-contiguous float64 numpy array")
    return a.ctypes.data_as(_dp)


class Context:
    """One device + one CUDA stream (w1mg_ctx)."""

    def __init__(self, device: int = 0):
        self.L = lib()
        h = C.c_void_p()
        check(self.L.w1mg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.L.w1mg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.L.w1mg_ctx_launch_count(self.h))

    @property
    def stream(self) -> int:
        return int(self.L.w1mg_ctx_stream(self.h) or 0)

    def level_seconds(self, levels: int):
        out = np.zeros(levels)
        n = self.L.w1mg_ctx_level_seconds(self.h, ptr(out), levels)
        if n < 0:
            check(-n)
        return out[:n].tolist()

    def synchronize(self):
        check(self.L.w1mg_ctx_synchronize(self.h))


_ctx = {}


def default_context(device: int = 0) -> Context:
    with _lock:
        c = _ctx.get(device)
    if c is None:
        c = Context(device)
        with _lock:
            _ctx[device] = c
    return c
