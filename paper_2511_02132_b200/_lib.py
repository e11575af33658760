"""ctypes loader for lib/libattnnuma.so (the C-ABI of include/attn_numa.h).

Argument marshalling only.  Fails loudly if the library is missing: there is
no fallback implementation anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ATTN_NUMA_LIB") or os.path.join(_PKG, "lib", "libattnnuma.so")

ATTN_MAX_DOMAINS = 8
ATTN_MAX_SMID = 512

# every symbol include/attn_numa.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "attn_fwd", "attn_fwd_stream", "attn_fwd_lse", "attn_bwd", "attn_fwd_host", "attn_bwd_host", "attn_set_stream", "attn_init", "attn_topology",
    "attn_set_topology_override", "attn_set_schedule_trace", "attn_schedule_order",
    "attn_last_launch_info", "attn_status_string", "attn_last_error", "attn_version", "attn_shutdown",
    "attn_fwd_replicated", "attn_ipc_get_handle", "attn_ipc_open", "attn_ipc_close", "attn_shf_acc_shared",
)


class Topology(ctypes.Structure):
    _fields_ = [
        ("num_sms", ctypes.c_int),
        ("nsmid", ctypes.c_int),
        ("n_domains", ctypes.c_int),
        ("sms_per_domain", ctypes.c_int * ATTN_MAX_DOMAINS),
        ("domain_of_smid", ctypes.c_byte * ATTN_MAX_SMID),
        ("lat_near_cyc", ctypes.c_float),
        ("lat_far_cyc", ctypes.c_float),
        ("far_lines_cached_near", ctypes.c_int),
        ("l2_bytes", ctypes.c_longlong),
        ("source", ctypes.c_int),
        ("stable", ctypes.c_int),
        ("lat_near_reread_cyc", ctypes.c_float),
        ("lat_far_reread_cyc", ctypes.c_float),
    ]


class TraceRec(ctypes.Structure):
    _fields_ = [
        ("b", ctypes.c_int32), ("h", ctypes.c_int32), ("unit", ctypes.c_int32),
        ("smid", ctypes.c_int32), ("domain", ctypes.c_int32), ("queue", ctypes.c_int32),
        ("stolen", ctypes.c_int32), ("seq", ctypes.c_int32), ("t_pop_ns", ctypes.c_uint64),
    ]


class LaunchInfo(ctypes.Structure):
    _fields_ = [("grid", ctypes.c_int), ("block", ctypes.c_int), ("smem_bytes", ctypes.c_int),
                ("units", ctypes.c_int), ("n_queues", ctypes.c_int), ("kernel_launches", ctypes.c_int),
                ("shf_acc_shared", ctypes.c_int)]


class IpcHandle(ctypes.Structure):
    _fields_ = [("handle", ctypes.c_ubyte * 64), ("offset", ctypes.c_longlong)]


_lib = None


def load():
    """Load (once) and type the library.  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2511_02132_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, f32, ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_longlong
    fwd_args = [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, f32, i32]
    lib.attn_fwd.argtypes = fwd_args
    lib.attn_fwd_stream.argtypes = fwd_args + [vp]
    lib.attn_fwd_host.argtypes = fwd_args + [vp]
    lib.attn_fwd_lse.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, f32, i32, vp]
    lib.attn_bwd.argtypes = [vp] * 9 + [i32, i32, i32, i32, i32, i32, f32, i32, vp]
    lib.attn_bwd_host.argtypes = [vp] * 9 + [i32, i32, i32, i32, i32, i32, f32, i32, vp]
    lib.attn_set_stream.argtypes = [vp]
    lib.attn_init.argtypes = [i32]
    lib.attn_topology.argtypes = [i32, ctypes.POINTER(Topology)]
    lib.attn_set_topology_override.argtypes = [i32, vp, i32, i32]
    lib.attn_set_schedule_trace.argtypes = [i32, vp, ll]
    lib.attn_schedule_order.argtypes = [i32, i32, i32, i32, i32, i32, vp, vp, ll, vp, vp]
    lib.attn_last_launch_info.argtypes = [ctypes.POINTER(LaunchInfo)]
    lib.attn_fwd_replicated.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, f32, i32, vp]
    lib.attn_ipc_get_handle.argtypes = [vp, ctypes.POINTER(IpcHandle)]
    lib.attn_ipc_open.argtypes = [ctypes.POINTER(IpcHandle), ctypes.POINTER(ctypes.c_void_p)]
    lib.attn_ipc_close.argtypes = [vp]
    lib.attn_shf_acc_shared.argtypes = [i32, i32, i32, ctypes.c_longlong]
    for f in ("attn_fwd", "attn_fwd_stream", "attn_fwd_lse", "attn_bwd", "attn_fwd_host", "attn_bwd_host", "attn_set_stream", "attn_init", "attn_topology",
              "attn_set_topology_override", "attn_set_schedule_trace", "attn_schedule_order",
              "attn_last_launch_info", "attn_fwd_replicated", "attn_ipc_get_handle", "attn_ipc_open",
              "attn_ipc_close", "attn_shf_acc_shared"):
        getattr(lib, f).restype = i32
    lib.attn_status_string.argtypes = [i32]
    lib.attn_status_string.restype = ctypes.c_char_p
    lib.attn_last_error.argtypes = []
    lib.attn_last_error.restype = ctypes.c_char_p
    lib.attn_version.argtypes = []
    lib.attn_version.restype = ctypes.c_char_p
    lib.attn_shutdown.argtypes = []
    lib.attn_shutdown.restype = None
    _lib = lib
    return lib
