"""ctypes binding of ``libwmpc.so`` (C ABI declared in ``include/wmpc.h``).

The library is built in-tree by ``paper_1904_10548_b200.build.build_native``
(called from ``__graft_entry__.build()``). There is no fallback: if the
library or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import weakref
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libwmpc.so")

WMPC_OK = 0
WMPC_E_ARG = -1
WMPC_E_CUDA = -2
WMPC_E_INFEASIBLE = -3
WMPC_E_NONFINITE = -4
WMPC_E_STATE = -5


class wmpc_dims(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64),
        ("horizon", C.c_int32),
        ("n_tanks", C.c_int32),
        ("n_inputs", C.c_int32),
        ("n_demands", C.c_int32),
        ("n_mixing", C.c_int32),
        ("device", C.c_int32),
    ]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)
_vp = C.c_void_p

# name -> (restype, argtypes)
SIGNATURES = {
    "wmpc_create": (C.c_int, [C.POINTER(wmpc_dims), C.POINTER(_vp)]),
    "wmpc_destroy": (None, [_vp]),
    "wmpc_last_error": (C.c_char_p, [_vp]),
    "wmpc_global_error": (C.c_char_p, []),
    "wmpc_set_structure": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _ip, _dp, _dp, _dp]),
    "wmpc_nodes_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "wmpc_nodes_destroy": (None, [_vp]),
    "wmpc_bind_nodes": (C.c_int, [_vp, _vp]),
    "wmpc_set_node_data": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp, _ip]),
    "wmpc_get_offsets": (C.c_int, [_vp, _vp, _dp, _dp]),
    "wmpc_set_bounds": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double, _dp, _dp, _dp]),
    "wmpc_dual_gradient": (C.c_int, [_vp, _dp, _dp, _dp]),
    "wmpc_prox": (C.c_int, [_vp, _dp, C.c_double, C.c_int, _dp]),
    "wmpc_power_iteration": (C.c_int, [_vp, _dp, C.c_double, C.c_int, _dp, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int)]),
    "wmpc_operator_trace": (C.c_int, [_vp, _dp]),
    "wmpc_apg_begin": (C.c_int, [_vp, C.c_double, C.c_int, _dp, _dp]),
    "wmpc_apg_run": (C.c_int, [_vp, C.c_int]),
    "wmpc_apg_warm": (C.c_int, [_vp, _dp]),
    "wmpc_set_precision": (C.c_int, [_vp, C.c_int]),
    "wmpc_apg_run_timed": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_float)]),
    "wmpc_iteration_profile": (C.c_int, [_vp, C.c_int, _dp, C.c_int]),
    "wmpc_apg_check": (C.c_int, [_vp, _dp, _dp, _dp, C.POINTER(C.c_int)]),
    "wmpc_certificate": (C.c_int, [_vp, _dp, _dp]),
    "wmpc_apg_read": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp, _dp]),
    "wmpc_apg_read_async": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp, _dp]),
    "wmpc_apg_read_wait": (C.c_int, [_vp]),
    "wmpc_apg_iterations": (C.c_int, [_vp]),
    "wmpc_kernel_launches_per_iteration": (C.c_int, [_vp]),
    "wmpc_fast_path": (C.c_int, [_vp]),
    "wmpc_path_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.c_int]),
    "wmpc_set_pdl": (C.c_int, [_vp, C.c_int]),
    "wmpc_profile_fast": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_uint64), C.c_int]),
    "wmpc_last_debug_ms": (C.c_float, [_vp]),
    "wmpc_debug_div": (C.c_int, [_dp, _dp, C.c_int, C.POINTER(C.c_uint64)]),
    "wmpc_timer_start": (C.c_int, [_vp]),
    "wmpc_timer_stop": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "wmpc_launch_count": (C.c_int64, [_vp]),
    "wmpc_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(_vp)]),
    "wmpc_host_free": (None, [_vp]),
    "wmpc_shard_setup": (C.c_int, [_vp, C.c_int, C.c_int, _ip, _ip]),
    "wmpc_shard_set_exchange": (C.c_int, [_vp, _vp]),
    "wmpc_shard_step": (C.c_int, [_vp, C.c_int]),
    "wmpc_sync": (C.c_int, [_vp]),
    "wmpc_nccl_unique_id": (C.c_int, [_vp]),
    "wmpc_shard_nccl_init": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "wmpc_shard_exchange": (C.c_int, [_vp]),
    "wmpc_set_min_branch_stage": (C.c_int, [_vp, C.c_int]),
    "wmpc_shard_fix_R": (C.c_int, [_vp, C.c_int]),
    "wmpc_cert_absmax": (C.c_int, [_vp, _dp]),
    "wmpc_cert_dykstra": (C.c_int, [_vp, C.c_int, _dp]),
    "wmpc_shard_dual_eval": (C.c_int, [_vp, C.c_int]),
    "wmpc_cert_terms": (C.c_int, [_vp, C.c_int, _dp]),
    "wmpc_u0_rows": (None, [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]),
}

_LIB = None


def load() -> C.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("WMPC_LIB_EXPERIMENT") or LIB_PATH  # A/B builds in tools/ only
        if not os.path.exists(path):
            raise RuntimeError(
                f"native library missing: {path}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    if a.dtype == np.int64:
        return a.ctypes.data_as(_ip)
    return a.ctypes.data_as(_dp)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class NativeError(RuntimeError):
    pass


PATH_FIELDS = ("fast_path", "fused_dp", "chainw", "ring_depth", "branch_groups", "nchain", "kstar",
               "ell_vf", "fp32", "dp_wpc", "dp_grid", "dp_cpw", "kernels_per_iteration", "n_branch", "sms",
               "dp_sib", "dp_segm")


def path_info(ctx: "Context") -> dict:
    """Kernel selection of the context's structure (wmpc_path_info)."""
    buf = (C.c_int * 32)()
    n = load().wmpc_path_info(ctx.h, buf, 32)
    return {k: int(buf[i]) for i, k in enumerate(PATH_FIELDS[:max(n, 0)])}


class Context:
    """Owns one ``wmpc_ctx`` (device buffers for one tree size)."""

    def __init__(self, n, horizon, n_tanks, n_inputs, n_demands, n_mixing, device=0):
        self.lib = load()
        dims = wmpc_dims(n, horizon, n_tanks, n_inputs, n_demands, n_mixing, device)
        h = _vp()
        rc = self.lib.wmpc_create(C.byref(dims), C.byref(h))
        if rc != WMPC_OK:
            msg = self.lib.wmpc_global_error().decode()
            if rc == WMPC_E_ARG:
                raise ValueError(msg)
            raise NativeError(f"wmpc_create failed: {msg}")
        self.h = h
        self.dims = (n, horizon, n_tanks, n_inputs, n_demands, n_mixing)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                self.lib.wmpc_destroy(h)
            except Exception:
                pass
            self.h = None

    def err(self) -> str:
        return self.lib.wmpc_last_error(self.h).decode()

    def call(self, name, *args):
        rc = getattr(self.lib, name)(self.h, *args)
        if rc == WMPC_OK:
            return
        msg = self.err()
        if rc in (WMPC_E_ARG, WMPC_E_INFEASIBLE):
            raise ValueError(msg)
        raise NativeError(f"{name}: {msg}")


class NodeSet:
    """Owns one ``wmpc_nodes`` (per-node factor state) of a context."""

    def __init__(self, ctx: Context):
        self.ctx = ctx  # keeps the context alive
        h = _vp()
        ctx.call("wmpc_nodes_create", C.byref(h))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                self.ctx.lib.wmpc_nodes_destroy(h)
            except Exception:
                pass
            self.h = None


class _Pinned:
    def __init__(self, nbytes):
        self.lib = load()
        p = _vp()
        if self.lib.wmpc_host_alloc(nbytes, C.byref(p)) != WMPC_OK:
            raise NativeError(self.lib.wmpc_global_error().decode())
        self.p = p

    def __del__(self):
        if getattr(self, "p", None):
            self.lib.wmpc_host_free(self.p)
            self.p = None


def pinned_copy(a) -> np.ndarray:
    """Copy of ``a`` in page-locked host memory (keeps its buffer alive)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    buf = _Pinned(max(a.nbytes, 8))
    raw = (C.c_double * max(a.size, 1)).from_address(buf.p.value)
    # every array or view over the block keeps `raw` alive; the block is
    # freed with the last of them (no id-keyed registry: ADVICE r1)
    weakref.finalize(raw, _free_pinned, buf)
    out = np.frombuffer(raw, dtype=np.float64, count=a.size).reshape(a.shape)
    out[...] = a
    return out


def _free_pinned(buf) -> None:
    buf.__del__()


class _PinnedPool:
    """Page-locked result arrays, recycled: a block returns to the pool when
    the last array (or view) over it is gone, so a caller that drops each
    solve's results reuses the same blocks instead of paying for page
    locking every solve."""

    def __init__(self, keep: int = 8):
        self.keep = keep
        self.free: dict = {}

    def empty(self, n: int) -> np.ndarray:
        nbytes = 8 * max(int(n), 1)
        lst = self.free.get(nbytes)
        buf = lst.pop() if lst else _Pinned(nbytes)
        raw = (C.c_double * max(int(n), 1)).from_address(buf.p.value)
        # every array or view over the block keeps `raw` alive
        weakref.finalize(raw, self._give, nbytes, buf)
        return np.frombuffer(raw, dtype=np.float64, count=int(n))

    def _give(self, nbytes, buf):
        lst = self.free.setdefault(nbytes, [])
        if len(lst) < self.keep:
            lst.append(buf)


_POOL = _PinnedPool()


def pinned_empty(n: int) -> np.ndarray:
    """Uninitialised float64 array of ``n`` elements in page-locked memory (pooled)."""
    return _POOL.empty(n)
