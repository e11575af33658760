"""Python binding of the C-ABI (include/attn_numa.h), same names.

Argument marshalling only: every step of the attention forward runs in the
CUDA kernels of lib/libattnnuma.so.  torch supplies device memory and the
current stream; nothing here computes attention.
"""
from __future__ import annotations

import ctypes
import math
from typing import Dict, List, Optional, Sequence

import torch

from . import _lib

MAPPINGS = {"block_first": 0, "head_first": 1, "swizzled_head_first": 2, "swizzled_block_first": 3,
            "bf": 0, "hf": 1, "shf": 2, "sbf": 3}
MAPPING_NAMES = ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first")


class AttnError(RuntimeError):
    def __init__(self, status: int, detail: str):
        lib = _lib.load()
        name = lib.attn_status_string(status).decode()
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.detail = detail


def _check(rc: int) -> None:
    if rc != 0:
        raise AttnError(rc, _lib.load().attn_last_error().decode())


ORDER_DESCENDING = 0x100  # include/attn_numa.h ATTN_ORDER_DESCENDING
CLUSTER_MULTICAST = 0x200  # include/attn_numa.h ATTN_CLUSTER_MULTICAST
ORDER_ALTERNATE = 0x400  # include/attn_numa.h ATTN_ORDER_ALTERNATE
ORDERS = {"ascending": 0, "descending": ORDER_DESCENDING, "alternate": ORDER_ALTERNATE}
SHF_ACC_SHARED = 0x800  # include/attn_numa.h ATTN_SHF_ACC_SHARED
SHF_ACC_PER_DIE = 0x1000  # include/attn_numa.h ATTN_SHF_ACC_PER_DIE
# "swizzled_head_first:shared" / ":per_die" force the SHF ACC grain (R23); no suffix = library rule
SHF_ACC = {"": 0, "shared": SHF_ACC_SHARED, "per_die": SHF_ACC_PER_DIE}
BWD_DETERMINISTIC = 0x2000  # include/attn_numa.h ATTN_BWD_DETERMINISTIC (two-pass backward, reproducible dq)


def _mapping_id(mapping, order: str = "ascending", cluster: bool = False) -> int:
    if isinstance(mapping, int):
        m = mapping
    else:
        name, _, grain = str(mapping).lower().partition(":")
        if grain not in SHF_ACC:
            raise ValueError("mapping suffix must be ':shared' or ':per_die'")
        m = MAPPINGS[name] | SHF_ACC[grain]
    if order not in ORDERS:
        raise ValueError("order must be 'ascending', 'descending' or 'alternate'")
    m |= ORDERS[order]
    if cluster:
        m |= CLUSTER_MULTICAST
    return m


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_tensor(name: str, t, shape, dtype=torch.bfloat16, cuda: bool = True) -> None:
    """One tensor against the C-ABI layout: contiguous, `dtype`, exactly
    `shape`, and on a CUDA device (cuda=True) or in host memory (cuda=False).
    The library sizes every copy and TMA view from q's shape, so a smaller or
    strided tensor would be read or written past its end."""
    where = "CUDA" if cuda else "CPU"
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or bool(t.is_cuda) != cuda:
        raise TypeError(f"{name} must be a {dtype} {where} tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (row-major {list(shape)})")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {list(t.shape)}, expected {list(shape)}")


def _qkv_shape(q, k, v, cuda: bool = True):
    """Validate q [B, Hq, N, d], k and v [B, Hkv, N, d] (same B, N, d); returns (B, Hq, Hkv, N, d)."""
    if not isinstance(q, torch.Tensor) or q.dim() != 4:
        raise ValueError("q must be a [B, Hq, N, d] tensor")
    if not isinstance(k, torch.Tensor) or k.dim() != 4:
        raise ValueError("k must be a [B, Hkv, N, d] tensor")
    B, Hq, N, d = q.shape
    Hkv = k.shape[1]
    _check_tensor("q", q, (B, Hq, N, d), cuda=cuda)
    _check_tensor("k", k, (B, Hkv, N, d), cuda=cuda)
    _check_tensor("v", v, (B, Hkv, N, d), cuda=cuda)
    if cuda and not (k.device == q.device and v.device == q.device):
        raise ValueError("q, k, v must be on one device")
    return B, Hq, Hkv, N, d


def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: Optional[torch.Tensor] = None, *,
             causal: bool = False, scale: Optional[float] = None, mapping="swizzled_head_first",
             order: str = "ascending", stream: Optional[torch.cuda.Stream] = None,
             cluster: bool = False) -> torch.Tensor:
    """O = softmax(scale * Q K^T) V (PAPER.md eq:fa) on bf16 [B, H, N, d] CUDA tensors.

    q: [B, Hq, N, d]; k, v: [B, Hkv, N, d]; returns o [B, Hq, N, d] (allocated
    if not given).  scale defaults to 1/sqrt(d).  Asynchronous on `stream`
    (default: torch's current stream).  `order` = "descending" visits each
    head's work units longest-first (ATTN_ORDER_DESCENDING); `cluster` runs
    CTA pairs that multicast K/V (ATTN_CLUSTER_MULTICAST).  Results are
    bit-identical either way.
    """
    B, Hq, Hkv, N, d = _qkv_shape(q, k, v)
    if o is None:
        o = torch.empty_like(q)
    else:
        _check_tensor("o", o, q.shape)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    lib = _lib.load()
    _check(lib.attn_fwd_stream(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), B, Hq, Hkv, N, d,
                               int(bool(causal)), float(scale), _mapping_id(mapping, order, cluster),
                               _stream_ptr(stream)))
    return o


def attn_fwd_replicated(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o_dst: Sequence, Hq_out: int,
                        head_offset: int, *, causal: bool = False, scale: Optional[float] = None,
                        mapping="swizzled_head_first", order: str = "ascending",
                        stream: Optional[torch.cuda.Stream] = None, cluster: bool = False) -> None:
    """Head-shard forward whose epilogue stores O into every destination (C-ABI attn_fwd_replicated).

    q/k/v: this rank's shard; o_dst: full [B, Hq_out, N, d] outputs, given as
    bf16 CUDA tensors (this device) or raw device addresses (peer buffers
    mapped with ipc_open).  The shard's heads land at head_offset."""
    B, Hq, Hkv, N, d = _qkv_shape(q, k, v)
    if not 1 <= len(o_dst) <= 8:
        raise ValueError("1 to 8 destinations")
    ptrs = []
    for t in o_dst:
        if isinstance(t, torch.Tensor):
            _check_tensor("o_dst[i]", t, (B, int(Hq_out), N, d))
            ptrs.append(t.data_ptr())
        else:
            ptrs.append(int(t))
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    lib = _lib.load()
    _check(lib.attn_fwd_replicated(q.data_ptr(), k.data_ptr(), v.data_ptr(), arr, len(ptrs), int(Hq_out),
                                   int(head_offset), B, Hq, Hkv, N, d, int(bool(causal)), float(scale),
                                   _mapping_id(mapping, order, cluster), _stream_ptr(stream)))


def ipc_get_handle(t: torch.Tensor) -> bytes:
    """72-byte CUDA IPC record (handle + offset) for a CUDA tensor's storage (C-ABI attn_ipc_get_handle)."""
    h = _lib.IpcHandle()
    _check(_lib.load().attn_ipc_get_handle(t.data_ptr(), ctypes.byref(h)))
    return bytes(h)


def ipc_open(record: bytes) -> int:
    """Map another process's ipc_get_handle record on the current device; returns the device address."""
    h = _lib.IpcHandle.from_buffer_copy(record)
    p = ctypes.c_void_p()
    _check(_lib.load().attn_ipc_open(ctypes.byref(h), ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(_lib.load().attn_ipc_close(ctypes.c_void_p(ptr)))


def attn_fwd_lse(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, causal: bool = False,
                 scale: Optional[float] = None, mapping="swizzled_head_first", order: str = "ascending",
                 stream: Optional[torch.cuda.Stream] = None, cluster: bool = False):
    """Forward that also returns the fp32 row log-sum-exp [B, Hq, N] (backward input)."""
    B, Hq, Hkv, N, d = _qkv_shape(q, k, v)
    o = torch.empty_like(q)
    lse = torch.empty((B, Hq, N), dtype=torch.float32, device=q.device)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    lib = _lib.load()
    _check(lib.attn_fwd_lse(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), B, Hq,
                            Hkv, N, d, int(bool(causal)), float(scale), _mapping_id(mapping, order, cluster),
                            _stream_ptr(stream)))
    return o, lse


def attn_bwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor, dout: torch.Tensor,
             lse: torch.Tensor, *, causal: bool = False, scale: Optional[float] = None,
             mapping="swizzled_head_first", order: str = "ascending", stream: Optional[torch.cuda.Stream] = None,
             dq: Optional[torch.Tensor] = None, dk: Optional[torch.Tensor] = None, dv: Optional[torch.Tensor] = None,
             deterministic: bool = False):
    """Gradients (dq, dk, dv) of sum(dout * attention(q, k, v)) (PAPER.md eq:ba), bf16.
    dq / dk / dv may be passed as preallocated outputs (shaped like q / k / v).
    deterministic=True selects the two-pass backward (bit-reproducible dq) for
    d <= 64, where the default single-pass kernel adds dq in arrival order."""
    B, Hq, Hkv, N, d = _qkv_shape(q, k, v)
    _check_tensor("o", o, q.shape)
    _check_tensor("dout", dout, q.shape)
    _check_tensor("lse", lse, (B, Hq, N), dtype=torch.float32)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    for name, t, ref in (("dq", dq, q), ("dk", dk, k), ("dv", dv, v)):
        _check_tensor(name, t, ref.shape)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    lib = _lib.load()
    _check(lib.attn_bwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                        dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), B, Hq, Hkv, N, d, int(bool(causal)),
                        float(scale), _mapping_id(mapping, order) | (BWD_DETERMINISTIC if deterministic else 0),
                        _stream_ptr(stream)))
    return dq, dk, dv


def attn_bwd_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor, dout: torch.Tensor,
                  lse: torch.Tensor, dq: torch.Tensor, dk: torch.Tensor, dv: torch.Tensor, *, causal: bool = False,
                  scale: Optional[float] = None, mapping="swizzled_head_first", order: str = "ascending",
                  stream: Optional[torch.cuda.Stream] = None, deterministic: bool = False):
    """End-to-end backward on HOST (ideally pinned) tensors: H2D of q, k, v, o,
    dout (bf16) and lse (fp32), the backward kernels, D2H of dq, dk, dv, sync.
    deterministic as attn_bwd."""
    B, Hq, Hkv, N, d = _qkv_shape(q, k, v, cuda=False)
    for name, t, shape in (("o", o, q.shape), ("dout", dout, q.shape), ("dq", dq, q.shape), ("dk", dk, k.shape),
                           ("dv", dv, k.shape)):
        _check_tensor(name, t, shape, cuda=False)
    _check_tensor("lse", lse, (B, Hq, N), dtype=torch.float32, cuda=False)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    lib = _lib.load()
    _check(lib.attn_bwd_host(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), dout.data_ptr(),
                             lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), B, Hq, Hkv, N, d,
                             int(bool(causal)), float(scale),
                             _mapping_id(mapping, order) | (BWD_DETERMINISTIC if deterministic else 0),
                             _stream_ptr(stream)))
    return dq, dk, dv


def attn_fwd_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor, *, causal: bool = False,
                  scale: Optional[float] = None, mapping="swizzled_head_first", order: str = "ascending",
                  stream: Optional[torch.cuda.Stream] = None, cluster: bool = False) -> torch.Tensor:
    """End-to-end call on HOST (ideally pinned) bf16 tensors: H2D, kernel, D2H, sync."""
    B, Hq, Hkv, N, d = _qkv_shape(q, k, v, cuda=False)
    _check_tensor("o", o, q.shape, cuda=False)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    lib = _lib.load()
    _check(lib.attn_fwd_host(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), B, Hq, Hkv, N, d,
                             int(bool(causal)), float(scale), _mapping_id(mapping, order, cluster),
                             _stream_ptr(stream)))
    return o


def attn_init(device: int = 0) -> None:
    _check(_lib.load().attn_init(int(device)))


def attn_topology(device: int = 0) -> Dict:
    t = _lib.Topology()
    _check(_lib.load().attn_topology(int(device), ctypes.byref(t)))
    return {
        "num_sms": t.num_sms, "nsmid": t.nsmid, "n_domains": t.n_domains,
        "sms_per_domain": list(t.sms_per_domain)[: max(t.n_domains, 1)],
        "domain_of_smid": list(t.domain_of_smid)[: t.nsmid],
        "lat_near_cyc": t.lat_near_cyc, "lat_far_cyc": t.lat_far_cyc,
        "far_lines_cached_near": t.far_lines_cached_near, "l2_bytes": t.l2_bytes,
        "lat_near_reread_cyc": t.lat_near_reread_cyc, "lat_far_reread_cyc": t.lat_far_reread_cyc,
        "source": ("probe", "override", "fallback")[t.source] if 0 <= t.source <= 2 else t.source,
        "stable": bool(t.stable),
    }


def attn_set_topology_override(device: int, domain_of_smid: Optional[Sequence[int]], n_domains: int = 2) -> None:
    lib = _lib.load()
    if domain_of_smid is None:
        _check(lib.attn_set_topology_override(int(device), None, 0, 0))
        return
    arr = (ctypes.c_byte * len(domain_of_smid))(*[int(x) for x in domain_of_smid])
    _check(lib.attn_set_topology_override(int(device), ctypes.cast(arr, ctypes.c_void_p), len(domain_of_smid),
                                          int(n_domains)))


def attn_set_schedule_trace(device: int, buf: Optional[torch.Tensor]) -> None:
    """buf: a CUDA uint8/int tensor of capacity*sizeof(TraceRec) bytes, or None."""
    lib = _lib.load()
    if buf is None:
        _check(lib.attn_set_schedule_trace(int(device), None, 0))
        return
    cap = buf.numel() * buf.element_size() // ctypes.sizeof(_lib.TraceRec)
    _check(lib.attn_set_schedule_trace(int(device), buf.data_ptr(), cap))


TRACE_FIELDS = ("b", "h", "unit", "smid", "domain", "queue", "stolen", "seq")


def trace_buffer(n_units: int, device="cuda") -> torch.Tensor:
    rec = ctypes.sizeof(_lib.TraceRec)
    return torch.full((n_units * rec // 4,), -1, dtype=torch.int32, device=device)


def decode_trace(buf: torch.Tensor) -> torch.Tensor:
    """[n_units, 8] int32 view (b, h, unit, smid, domain, queue, stolen, seq); t_pop dropped."""
    rec_words = ctypes.sizeof(_lib.TraceRec) // 4
    return buf.view(-1, rec_words)[:, :8].cpu()


def attn_schedule_order(B: int, Hq: int, Hkv: int, N: int, mapping, sms_per_domain: Sequence[int],
                        order: str = "ascending", cluster: bool = False) -> List[List[tuple]]:
    """Host-side queues (lists of (b, h, unit)) the kernel would pop (unit = 256 rows)."""
    lib = _lib.load()
    U = (N + 255) // 256
    cap = B * Hq * U
    out = (ctypes.c_int32 * (3 * cap))()
    nq = ctypes.c_int(0)
    qlen = (ctypes.c_int * _lib.ATTN_MAX_DOMAINS)()
    sizes = (ctypes.c_int * len(sms_per_domain))(*sms_per_domain)
    _check(lib.attn_schedule_order(B, Hq, Hkv, N, _mapping_id(mapping, order, cluster), len(sms_per_domain),
                                   ctypes.cast(sizes, ctypes.c_void_p), ctypes.cast(out, ctypes.c_void_p), cap,
                                   ctypes.cast(ctypes.pointer(nq), ctypes.c_void_p),
                                   ctypes.cast(qlen, ctypes.c_void_p)))
    flat = list(out)
    queues, w = [], 0
    for qi in range(nq.value):
        q = []
        for _ in range(qlen[qi]):
            q.append((flat[3 * w], flat[3 * w + 1], flat[3 * w + 2]))
            w += 1
        queues.append(q)
    return queues


def attn_shf_acc_shared(n_domains: int, N: int, d: int, l2_bytes: int) -> bool:
    """The library's SHF ACC-grain rule (C-ABI attn_shf_acc_shared, R23)."""
    return bool(_lib.load().attn_shf_acc_shared(n_domains, N, d, l2_bytes))


def attn_last_launch_info() -> Dict:
    info = _lib.LaunchInfo()
    _check(_lib.load().attn_last_launch_info(ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in _lib.LaunchInfo._fields_}


def attn_version() -> str:
    return _lib.load().attn_version().decode()


def attn_shutdown() -> None:
    _lib.load().attn_shutdown()
