"""B200-native Swizzled-Head-first attention forward (arxiv 2511.02132 hot path).

The compute path is lib/libattnnuma.so (C-ABI, include/attn_numa.h): an
sm_100a tcgen05/TMEM/TMA FlashAttention-2-style forward kernel whose work
units are handed to SMs by a persistent scheduler in block-first, head-first
or swizzled head-first order.  This package is a thin ctypes binding.
"""
from .api import (AttnError, MAPPING_NAMES, MAPPINGS, attn_bwd, attn_bwd_host, attn_fwd, attn_fwd_host, attn_fwd_lse, attn_fwd_replicated,
                  attn_init, ipc_close, ipc_get_handle, ipc_open,
                  attn_last_launch_info, attn_schedule_order, attn_set_schedule_trace, attn_shf_acc_shared,
                  attn_set_topology_override, attn_shutdown, attn_topology, attn_version,
                  decode_trace, trace_buffer)

__all__ = [
    "AttnError", "MAPPINGS", "MAPPING_NAMES", "attn_bwd", "attn_bwd_host", "attn_fwd", "attn_fwd_host", "attn_fwd_lse", "attn_fwd_replicated", "attn_init", "ipc_close",
    "ipc_get_handle", "ipc_open",
    "attn_last_launch_info", "attn_schedule_order", "attn_set_schedule_trace", "attn_shf_acc_shared",
    "attn_set_topology_override", "attn_shutdown", "attn_topology", "attn_version",
    "decode_trace", "trace_buffer",
]
