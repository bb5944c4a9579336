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
        ("has_label_scale", ctypes.c_int32), ("label_scale", ctypes.c_double * 9),
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


class HostCsr(ctypes.Structure):
    _fields_ = [("arena", ctypes.c_void_p), ("nnz", ctypes.c_int64), ("off_indptr", ctypes.c_int64),
                ("off_indices", ctypes.c_int64), ("off_data", ctypes.c_int64)]


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
    "nlg_assemble_pinned": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ALLOC_FN,
                                             ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(Stats),
                                             ctypes.POINTER(HostCsr)]),
    "nlg_pinned_alloc": (ctypes.c_void_p, [ctypes.c_int64]),
    "nlg_pinned_free": (None, [ctypes.c_void_p]),
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


class PinnedPool:
    """Page-locked host blocks for host-resident CSR outputs (nlg_assemble_pinned).

    Pinning memory costs ~0.2 s per GB, so blocks are recycled: a block goes
    back to the pool when the last numpy view of it is collected, and the
    next assembly of a similar size takes it again.  The ``keep`` most recently
    returned blocks (NLG_PINNED_KEEP, default 2) stay pinned; older ones are released.
    """

    _GRAIN = 1 << 26  # 64 MiB: similar sizes share a block

    def __init__(self):
        self._free = []  # (capacity, address)
        self._mu = threading.Lock()
        self.keep = int(os.environ.get("NLG_PINNED_KEEP", "2"))
        self.n_alloc = 0

    def take(self, nbytes):
        """(address, capacity) of a block of at least nbytes, or (None, 0)."""
        need = max(int(nbytes), 1)
        with self._mu:
            fit = [b for b in self._free if need <= b[0] <= 2 * need + self._GRAIN]
            if fit:
                blk = min(fit)
                self._free.remove(blk)
                return blk[1], blk[0]
        cap = (need + self._GRAIN - 1) // self._GRAIN * self._GRAIN
        addr = load_library().nlg_pinned_alloc(cap)
        if not addr:
            self.trim(0)  # release what is pooled and retry once
            addr = load_library().nlg_pinned_alloc(cap)
            if not addr:
                return None, 0
        self.n_alloc += 1
        return int(addr), cap

    def give(self, addr, cap):
        with self._mu:
            self._free.append((cap, addr))
        self.trim(self.keep)

    def trim(self, keep):
        with self._mu:  # (least recently returned first)
            cut = max(len(self._free) - keep, 0)
            drop, self._free = self._free[:cut], self._free[cut:]
        lib = _lib
        for _, addr in drop:
            if lib is not None:
                lib.nlg_pinned_free(ctypes.c_void_p(addr))

    def view(self, addr, cap):
        """uint8 numpy array over the block; the block returns to the pool
        when the array and every view of it are gone."""
        import weakref
        raw = (ctypes.c_ubyte * cap).from_address(addr)
        weakref.finalize(raw, self.give, addr, cap)
        return np.frombuffer(raw, dtype=np.uint8)


PINNED = PinnedPool()


class PinnedSink:
    """Block callback of nlg_assemble_pinned: hands out pooled page-locked
    blocks and turns the one the library used into the CSR arrays.  When no
    page-locked memory can be had (host limits), the block is ordinary numpy
    memory: the library's copies still land there, only slower."""

    def __init__(self):
        self.blocks = []  # (address, capacity, owner) handed out during this call; owner: numpy fallback
        self._cb = ALLOC_FN(self._alloc)

    def _alloc(self, user, nbytes, which):
        try:
            addr, cap = PINNED.take(nbytes)
            owner = None
            if addr is None:
                owner = np.empty(max(int(nbytes), 8), dtype=np.uint8)
                addr, cap = int(owner.ctypes.data), owner.size
            self.blocks.append((addr, cap, owner))
            return addr
        except Exception:  # noqa: BLE001 -- NULL makes the library fail cleanly
            return None

    @property
    def callback(self):
        return self._cb

    def release(self, keep_addr=None):
        """Blocks not holding the result go back to the pool; the result's
        (address, capacity, owner) is returned."""
        kept = None
        for addr, cap, owner in self.blocks:
            if keep_addr is not None and addr == keep_addr and kept is None:
                kept = (addr, cap, owner)
            elif owner is None:
                PINNED.give(addr, cap)
        self.blocks = []
        return kept

    def arrays(self, out, n_rows):
        kept = self.release(out.arena)
        if kept is None:
            raise DeviceError("nlg_assemble_pinned returned a block this sink did not hand out")
        buf = kept[2] if kept[2] is not None else PINNED.view(kept[0], kept[1])
        nnz = int(out.nnz)
        indptr = buf[out.off_indptr:out.off_indptr + 8 * (n_rows + 1)].view(np.int64)
        indices = buf[out.off_indices:out.off_indices + 4 * nnz].view(np.int32)
        data = buf[out.off_data:out.off_data + 8 * nnz].view(np.float64)
        return indptr, indices, data
