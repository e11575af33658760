"""The Python binding validates every tensor against the C-ABI layout before
calling the library: the library sizes its TMA views and host
copies from q's shape, so an undersized, strided or mistyped tensor must be
rejected in Python.  These cases never reach the library (no GPU needed)."""
import pytest
import torch

from paper_2511_02132_b200 import api


def _host(*shape, dtype=torch.bfloat16):
    return torch.zeros(shape, dtype=dtype)


def test_fwd_host_rejects_undersized_output():
    q, k, v = _host(1, 4, 64, 64), _host(1, 2, 64, 64), _host(1, 2, 64, 64)
    with pytest.raises(ValueError):
        api.attn_fwd_host(q, k, v, _host(1, 4, 32, 64))


def test_fwd_host_rejects_mismatched_kv():
    q = _host(1, 4, 64, 64)
    with pytest.raises(ValueError):
        api.attn_fwd_host(q, _host(1, 2, 64, 64), _host(1, 2, 63, 64), _host(1, 4, 64, 64))
    with pytest.raises(ValueError):
        api.attn_fwd_host(q, _host(1, 2, 64, 32), _host(1, 2, 64, 32), _host(1, 4, 64, 64))


def test_fwd_host_rejects_strided_or_wrong_dtype():
    q = _host(1, 64, 4, 64).transpose(1, 2)  # [B, N, H, d] storage viewed as [B, H, N, d]
    k, v, o = _host(1, 4, 64, 64), _host(1, 4, 64, 64), _host(1, 4, 64, 64)
    with pytest.raises(ValueError):
        api.attn_fwd_host(q, k, v, o)
    with pytest.raises(TypeError):
        api.attn_fwd_host(_host(1, 4, 64, 64, dtype=torch.float16), k, v, o)


def test_bwd_host_checks_every_tensor():
    q, k, v = _host(1, 4, 64, 64), _host(1, 2, 64, 64), _host(1, 2, 64, 64)
    o, do = _host(1, 4, 64, 64), _host(1, 4, 64, 64)
    lse = _host(1, 4, 64, dtype=torch.float32)
    dq, dk, dv = _host(1, 4, 64, 64), _host(1, 2, 64, 64), _host(1, 2, 64, 64)
    bad = dict(o=_host(1, 4, 32, 64), dout=_host(1, 2, 64, 64), lse=_host(1, 4, 32, dtype=torch.float32),
               dq=_host(1, 2, 64, 64), dk=_host(1, 4, 64, 64), dv=_host(1, 2, 64, 32))
    args = dict(q=q, k=k, v=v, o=o, dout=do, lse=lse, dq=dq, dk=dk, dv=dv)
    for name, t in bad.items():
        a = dict(args, **{name: t})
        with pytest.raises(ValueError):
            api.attn_bwd_host(a["q"], a["k"], a["v"], a["o"], a["dout"], a["lse"], a["dq"], a["dk"], a["dv"])
    with pytest.raises(TypeError):
        api.attn_bwd_host(q, k, v, o, do, lse.double(), dq, dk, dv)


def test_device_entry_points_reject_host_tensors():
    q, k, v = _host(1, 2, 64, 64), _host(1, 2, 64, 64), _host(1, 2, 64, 64)
    for fn in (api.attn_fwd, api.attn_fwd_lse):
        with pytest.raises(TypeError):
            fn(q, k, v)
    with pytest.raises(TypeError):
        api.attn_bwd(q, k, v, q, q, _host(1, 2, 64, dtype=torch.float32))
    with pytest.raises(TypeError):
        api.attn_fwd_replicated(q, k, v, [0], 2, 0)
