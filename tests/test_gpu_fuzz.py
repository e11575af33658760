"""Randomised parity: seeded random shapes x mapping x unit order x cluster
multicast, each checked against the fp64 oracle on sampled rows (every edge
row of the ragged tail included) and bit-identical to the plain block-first
launch of the same inputs.  Complements the hand-picked shapes of
test_gpu_parity / test_gpu_cluster."""
import math
import os
import random

import numpy as np
import pytest
import torch

from oracle import attn as oa
from tolerance import check_grad
from paper_2511_02132_b200 import attn_bwd, attn_fwd, attn_fwd_lse, synth

from test_gpu_parity import MAX_TOL, MEAN_TOL

pytestmark = pytest.mark.gpu

MAPS = ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first", "swizzled_head_first:shared")


def _cases(n, seed):
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        Hkv = rng.choice([1, 2, 3, 4])
        G = rng.choice([1, 2, 4, 8])
        N = rng.choice([1, 7, 128, 129, 255, 256, 300, rng.randint(1, 1500)])
        out.append(dict(B=rng.randint(1, 3), Hq=Hkv * G, Hkv=Hkv, N=N, d=8 * rng.randint(1, 16),
                        causal=rng.random() < 0.5, mapping=rng.choice(MAPS),
                        order=rng.choice(["ascending", "descending"]), cluster=rng.random() < 0.5,
                        seed=rng.randint(0, 1 << 20)))
    return out


# ATTN_FUZZ_CASES / ATTN_FUZZ_SEED widen the forward fuzz for one-off runs
_N_FWD = int(os.environ.get("ATTN_FUZZ_CASES", "40"))
_SEED_FWD = int(os.environ.get("ATTN_FUZZ_SEED", "2511"))


@pytest.mark.parametrize("case", _cases(_N_FWD, _SEED_FWD), ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_forward_fuzz(case):
    B, Hq, Hkv, N, d, causal = case["B"], case["Hq"], case["Hkv"], case["N"], case["d"], case["causal"]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=case["seed"], device="cuda")
    o = torch.full_like(q, float("nan"))
    attn_fwd(q, k, v, o, causal=causal, mapping=case["mapping"], order=case["order"], cluster=case["cluster"])
    plain = attn_fwd(q, k, v, causal=causal, mapping="block_first")
    torch.cuda.synchronize()
    assert torch.equal(o.view(torch.int16), plain.view(torch.int16)), "differs bitwise from the plain path"
    rng = np.random.default_rng(case["seed"])
    idx = sorted({0, N - 1, max(0, N - 129), min(N - 1, 127), min(N - 1, 128)} |
                 set(rng.integers(0, N, size=min(N, 24)).tolist()))
    rows = np.array([(int(rng.integers(B)), int(rng.integers(Hq)), i) for i in idx], dtype=np.int64)
    ref = oa.attention_rows(q.cpu(), k.cpu(), v.cpu(), rows, causal=causal, scale=1.0 / math.sqrt(d))
    got = o[rows[:, 0], rows[:, 1], rows[:, 2]].float().cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    assert np.isfinite(got).all() and err.max() <= MAX_TOL and err.mean() <= MEAN_TOL, (err.max(), err.mean())


_N_BWD = int(os.environ.get("ATTN_FUZZ_BWD_CASES", "12"))


@pytest.mark.parametrize("case", [c for c in _cases(_N_BWD, _SEED_FWD if _N_BWD != 12 else 77) if c["N"] <= 700],
                         ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_backward_fuzz(case):
    B, Hq, Hkv, N, d, causal = case["B"], case["Hq"], case["Hkv"], case["N"], case["d"], case["causal"]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=case["seed"], device="cuda")
    do = synth.make_tensor("q", B, Hq, N, d, base=case["seed"] + 1, device="cuda")
    o, lse = attn_fwd_lse(q, k, v, causal=causal)
    dq, dk, dv = attn_bwd(q, k, v, o, do, lse, causal=causal, mapping=case["mapping"], order=case["order"])
    torch.cuda.synchronize()
    rq, rk, rv, rl = oa.attention_bwd(q.cpu(), k.cpu(), v.cpu(), do.cpu(), causal=causal, scale=1.0 / math.sqrt(d))
    assert np.abs(lse.cpu().numpy() - rl).max() <= 1e-3
    for name, g, r in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv)):
        check_grad(f"{name} {case}", g, r)  # DESIGN.md reading R21 (tests/tolerance.py)
