"""ctypes wrapper over oracle/oracle_attn.c -- the fp64 CPU attention oracle.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package.  See oracle_attn.c for the definition it implements (PAPER.md:149-155
eq:fa, :167 MHA/GQA, :172, :187) and the readings R1-R5 it takes.

Inputs may be numpy arrays of dtype uint16 (raw bf16 bit patterns), float32 or
float64, or torch CPU tensors (bfloat16 / float32 / float64).  Outputs are
float64 numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_attn.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -fopenmp).  Returns the path."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", _SRC, "-o", _SO, "-lm"]
        )
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        common = [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, f64]
        lib.oracle_attn_full.argtypes = common + [vp]
        lib.oracle_attn_rows.argtypes = common + [vp, i64, vp]
        lib.oracle_attn_weights.argtypes = common + [i64, i64, i64, vp, vp]
        for f in (lib.oracle_attn_full, lib.oracle_attn_rows, lib.oracle_attn_weights):
            f.restype = i32
        lib.oracle_attn_bwd.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, f64, vp, vp, vp, vp]
        lib.oracle_attn_bwd.restype = i32
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_set_threads.restype = None
        lib.oracle_max_threads.argtypes = []
        lib.oracle_max_threads.restype = i32
        _lib = lib
    return _lib


def _as_np(x):
    """Return (contiguous numpy array, dtype code) without changing any value."""
    try:
        import torch

        if isinstance(x, torch.Tensor):
            x = x.detach().cpu().contiguous()
            if x.dtype == torch.bfloat16:
                return x.view(torch.int16).numpy().view(np.uint16), 0
            if x.dtype == torch.float32:
                return x.numpy(), 1
            if x.dtype == torch.float64:
                return x.numpy(), 2
            raise TypeError(f"unsupported torch dtype {x.dtype}")
    except ImportError:  # pragma: no cover
        pass
    x = np.ascontiguousarray(x)
    code = {np.dtype(np.uint16): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}.get(x.dtype)
    if code is None:
        raise TypeError(f"unsupported numpy dtype {x.dtype}")
    return x, code


def _prep(q, k, v):
    qa, cq = _as_np(q)
    ka, ck = _as_np(k)
    va, cv = _as_np(v)
    if not (cq == ck == cv):
        raise TypeError("q, k, v must share one element type")
    if qa.ndim != 4 or ka.ndim != 4 or va.ndim != 4:
        raise ValueError("expected [B, H, N, d] tensors")
    B, Hq, N, d = qa.shape
    Hkv = ka.shape[1]
    if ka.shape != (B, Hkv, N, d) or va.shape != ka.shape:
        raise ValueError("k, v must be [B, Hkv, N, d] matching q")
    return qa, ka, va, cq, (B, Hq, Hkv, N, d)


def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def attention(q, k, v, causal: bool = False, scale: float | None = None) -> np.ndarray:
    """Full fp64 attention, shape [B, Hq, N, d]."""
    qa, ka, va, code, (B, Hq, Hkv, N, d) = _prep(q, k, v)
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))  # eq:fa
    out = np.empty((B, Hq, N, d), dtype=np.float64)
    rc = _load().oracle_attn_full(qa.ctypes.data, ka.ctypes.data, va.ctypes.data, code,
                                  B, Hq, Hkv, N, d, int(bool(causal)), float(scale),
                                  out.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_attn_full failed ({rc})")
    return out


def attention_rows(q, k, v, rows, causal: bool = False, scale: float | None = None) -> np.ndarray:
    """fp64 attention for selected rows; rows is an (n, 3) int array of (b, h, i)."""
    qa, ka, va, code, (B, Hq, Hkv, N, d) = _prep(q, k, v)
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).reshape(-1, 3))
    out = np.empty((r.shape[0], d), dtype=np.float64)
    rc = _load().oracle_attn_rows(qa.ctypes.data, ka.ctypes.data, va.ctypes.data, code,
                                  B, Hq, Hkv, N, d, int(bool(causal)), float(scale),
                                  r.ctypes.data, r.shape[0], out.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_attn_rows failed ({rc})")
    return out


def attention_weights(q, k, v, b: int, h: int, i: int, causal: bool = False,
                      scale: float | None = None):
    """(normalised weights P[b,h,i,:] of length N, output row of length d)."""
    qa, ka, va, code, (B, Hq, Hkv, N, d) = _prep(q, k, v)
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))
    w = np.empty(N, dtype=np.float64)
    o = np.empty(d, dtype=np.float64)
    rc = _load().oracle_attn_weights(qa.ctypes.data, ka.ctypes.data, va.ctypes.data, code,
                                     B, Hq, Hkv, N, d, int(bool(causal)), float(scale),
                                     int(b), int(h), int(i), w.ctypes.data, o.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_attn_weights failed ({rc})")
    return w, o


def attention_bwd(q, k, v, dout, causal: bool = False, scale: float | None = None):
    """fp64 gradients (dq, dk, dv) of sum(dout * attention(q, k, v)) and the
    natural-log row LSE, per eq:ba.  O(N^2) memory per head:
    small shapes only."""
    qa, ka, va, code, (B, Hq, Hkv, N, d) = _prep(q, k, v)
    da, cd = _as_np(dout)
    if cd != code or da.shape != qa.shape:
        raise ValueError("dout must match q in shape and element type")
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))
    dq = np.empty((B, Hq, N, d), dtype=np.float64)
    dk = np.empty((B, Hkv, N, d), dtype=np.float64)
    dv = np.empty((B, Hkv, N, d), dtype=np.float64)
    lse = np.empty((B, Hq, N), dtype=np.float64)
    rc = _load().oracle_attn_bwd(qa.ctypes.data, ka.ctypes.data, va.ctypes.data, da.ctypes.data, code, B, Hq, Hkv, N,
                                 d, int(bool(causal)), float(scale), dq.ctypes.data, dk.ctypes.data, dv.ctypes.data,
                                 lse.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_attn_bwd failed ({rc})")
    return dq, dk, dv, lse


def _f64(a, code):
    """fp64 values of an _as_np array (bf16 bit patterns widened exactly)."""
    if code == 0:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def attention_bwd_rows(q, k, v, dout, b: int, g: int, q_rows, k_rows, causal: bool = False,
                       scale: float | None = None, chunk: int = 1024):
    """fp64 gradient ROWS of batch item b and KV head g per eq:ba,
    for sequences too long for attention_bwd's O(N^2) memory:
      dq[hh, r] = dq[b, g*G + hh, q_rows[r], :] for every query head of group g,
      dk[r], dv[r] = dk[b, g, k_rows[r], :], dv[b, g, k_rows[r], :].
    Step by step (numpy, not the C oracle), for each query head h of the group:
      1. over ALL query rows i, in chunks of `chunk` rows: s_ij = scale q_i.k_j
         (masked j > i when causal), lse_i = log sum_j exp(s_ij),
         o_i = sum_j exp(s_ij - lse_i) v_j, D_i = dO_i . o_i;
      2. P_ij = exp(s_ij - lse_i), dP_ij = dO_i . v_j, dS_ij = P_ij (dP_ij - D_i);
         dq_i = scale sum_j dS_ij k_j (sampled i);
         dv_j += sum_i P_ij dO_i,  dk_j += scale sum_i dS_ij q_i (sampled j;
         summed over the group's query heads)."""
    qa, ka, va, code, (B, Hq, Hkv, N, d) = _prep(q, k, v)
    da, cd = _as_np(dout)
    if cd != code or da.shape != qa.shape:
        raise ValueError("dout must match q in shape and element type")
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))
    G = Hq // Hkv
    qr = np.asarray(q_rows, dtype=np.int64)
    kr = np.asarray(k_rows, dtype=np.int64)
    K = _f64(ka[b, g], code)
    V = _f64(va[b, g], code)
    dq = np.zeros((G, len(qr), d))
    dk = np.zeros((len(kr), d))
    dv = np.zeros((len(kr), d))
    idx = np.arange(N)
    for hh in range(G):
        h = g * G + hh
        Q = _f64(qa[b, h], code)
        dO = _f64(da[b, h], cd)
        lse = np.empty(N)
        Dv = np.empty(N)
        for c0 in range(0, N, chunk):  # step 1: row statistics of every query row
            c1 = min(N, c0 + chunk)
            s = scale * (Q[c0:c1] @ K.T)
            if causal:
                s[idx[None, :] > idx[c0:c1, None]] = -np.inf
            m = s.max(axis=1)
            e = np.exp(s - m[:, None])
            l_ = e.sum(axis=1)
            lse[c0:c1] = m + np.log(l_)
            Dv[c0:c1] = (dO[c0:c1] * ((e @ V) / l_[:, None])).sum(axis=1)
        # step 2, sampled query rows: dq_i
        s = scale * (Q[qr] @ K.T)
        if causal:
            s[idx[None, :] > qr[:, None]] = -np.inf
        p = np.exp(s - lse[qr, None])
        ds = p * (dO[qr] @ V.T - Dv[qr, None])
        dq[hh] = scale * (ds @ K)
        # step 2, sampled key rows: dv_j, dk_j (column j of P over all queries)
        s = scale * (Q @ K[kr].T)
        if causal:
            s[kr[None, :] > idx[:, None]] = -np.inf
        p = np.exp(s - lse[:, None])
        dv += p.T @ dO
        ds = p * (dO @ V[kr].T - Dv[:, None])
        dk += scale * (ds.T @ Q)
    return dq, dk, dv
