"""ctypes binding of ``libnlg.so`` (the C ABI of include/nlg.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_2207_03921_b200.build``.  Loading fails loudly: there is
no CPU fallback for the assembly path.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import ConfigurationError, DeviceError, NumericalError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NLG_LIBRARY") or os.path.join(_HERE, "libnlg.so")

NLG_OK, NLG_ERR_CONFIG, NLG_ERR_NUMERICAL, NLG_ERR_CUDA = 0, 1, 2, 3

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)


class Problem(ctypes.Structure):
    _fields_ = [
        ("n_vertices", ctypes.c_int64), ("n_elements", ctypes.c_int64),
        ("vertices", ctypes.c_void_p), ("elements", ctypes.c_void_p),
        ("labels", ctypes.c_void_p), ("outer_mask", ctypes.c_void_p),
        ("dof_map", ctypes.c_void_p), ("n_dofs", ctypes.c_int64),
        ("nc", ctypes.c_int32), ("is_dg", ctypes.c_int32), ("kernel_id", ctypes.c_int32),
        ("ball_id", ctypes.c_int32), ("path_touch", ctypes.c_int32), ("symmetric", ctypes.c_int32),
        ("s", ctypes.c_double), ("scale", ctypes.c_double), ("delta", ctypes.c_double),
        ("rskip2", ctypes.c_double), ("drop2", ctypes.c_double),
        ("kp0", ctypes.c_double), ("kp1", ctypes.c_double),
        ("n_outer", ctypes.c_int32), ("n_inner", ctypes.c_int32),
        ("op", ctypes.c_void_p), ("ow", ctypes.c_void_p), ("oh", ctypes.c_void_p),
        ("ip", ctypes.c_void_p), ("iw", ctypes.c_void_p),
        ("n_sing", ctypes.c_int32 * 3),
        ("sxs", ctypes.c_void_p * 3), ("sys", ctypes.c_void_p * 3), ("sw", ctypes.c_void_p * 3),
        ("shx", ctypes.c_void_p * 3), ("shy", ctypes.c_void_p * 3),
        ("inputs_on_device", ctypes.c_int32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "n_roots", "epi", "n_full", "n_partial", "n_singular", "inner_evals", "outer_nonempty",
        "sing_points", "alg_flops", "alg_flops_full", "alg_flops_partial", "alg_flops_singular", "coo_entries", "coo_reduced", "nnz", "n_batches", "n_replans", "err_k", "err_l")] + [
        (n, ctypes.c_double) for n in (
            "ms_prep", "ms_candidates", "ms_full", "ms_partial", "ms_singular", "ms_merge",
            "ms_total", "ms_integrate_kernels", "ms_merge_stage_r")] + [
        (n, ctypes.c_int64) for n in ("n_row_retries", "n_merge_fallbacks", "err_self_k")]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32)

# symbols of include/nlg.h, with (restype, argtypes)
SIGNATURES = {
    "nlg_abi_version": (ctypes.c_int32, []),
    "nlg_last_error": (ctypes.c_char_p, []),
    "nlg_device_count": (ctypes.c_int32, [ctypes.POINTER(ctypes.c_int32)]),
    "nlg_plan_create": (ctypes.c_int32, [ctypes.c_int32, ctypes.POINTER(Problem), ctypes.c_void_p,
                                         ctypes.POINTER(ctypes.c_void_p)]),
    "nlg_plan_destroy": (None, [ctypes.c_void_p]),
    "nlg_assemble": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                      ALLOC_FN, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(Stats)]),
    "nlg_load_points": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, ALLOC_FN, ctypes.c_void_p,
                                         ctypes.POINTER(ctypes.c_int64)]),
    "nlg_load": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                  ALLOC_FN, ctypes.c_void_p]),
    "nlg_load_const": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ALLOC_FN,
                                        ctypes.c_void_p]),
    "nlg_mass": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, ALLOC_FN, ctypes.c_void_p]),
    "nlg_cg": (ctypes.c_int32, [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int32,
                                ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)]),
    "nlg_row_work": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_void_p]),
    "nlg_local_blocks": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "nlg_fp64_peak": (ctypes.c_int32, [ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]),
    "nlg_launch_count": (ctypes.c_int64, []),
    "nlg_last_batches": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]),
    "nlg_format_f64": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int32]),
    "nlg_format_i64": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int32]),
    "nlg_format_i32": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int32]),
}

_lib = None
_lock = threading.Lock()


def load_library(path=LIB_PATH):
    """Load libnlg.so and bind every symbol; raises DeviceError when absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is missing: build it with `python -m paper_2207_03921_b200.build` "
                "(there is no CPU fallback for the assembly path)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc, what="libnlg"):
    if rc == NLG_OK:
        return
    msg = load_library().nlg_last_error().decode(errors="replace")
    if rc == NLG_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == NLG_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise DeviceError(f"{what}: {msg}")


def device_count():
    n = ctypes.c_int32(0)
    load_library().nlg_device_count(ctypes.byref(n))
    return int(n.value)


def launch_count():
    return int(load_library().nlg_launch_count())


def fp64_peak_tflops(device=0):
    out = ctypes.c_double(0.0)
    check(load_library().nlg_fp64_peak(device, ctypes.byref(out)), "nlg_fp64_peak")
    return float(out.value)


class OutputSink:
    """Allocation callback target: numpy buffers (host) or torch tensors (device).

    ``reuse`` keeps the buffers of earlier calls and hands them out again when
    they are large enough (device outputs of repeated assemblies).
    """

    def __init__(self, on_host, device=0, reuse=None):
        self.on_host = on_host
        self.device = device
        self.bufs = {}
        self._pool = reuse if reuse is not None else {}
        self._cb = ALLOC_FN(self._alloc)

    def _alloc(self, user, nbytes, which):
        try:
            n = max(int(nbytes), 8)
            old = self._pool.get(which)
            if old is not None and old.numel() >= n and not self.on_host:
                self.bufs[which] = old
                return old.data_ptr()
            if self.on_host:
                buf = np.empty(n, dtype=np.uint8)
                self.bufs[which] = buf
                return buf.ctypes.data
            import torch
            buf = torch.empty((n + n // 8 + 15) // 16 * 16, dtype=torch.uint8, device=f"cuda:{self.device}")
            self.bufs[which] = buf
            self._pool[which] = buf
            return buf.data_ptr()
        except Exception:  # noqa: BLE001 -- returning NULL makes the library fail cleanly
            return None

    @property
    def callback(self):
        return self._cb

    def array(self, which, dtype, count):
        buf = self.bufs[which]
        if self.on_host:
            return buf.view(dtype)[:count]
        import torch
        tdt = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[np.dtype(dtype).type]
        return buf.view(tdt)[:count]
