"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/attn_numa.h declares, validates arguments synchronously (status codes
before any CUDA call), and its host-side queue builder reproduces the
mapping reference in oracle/mapping.py exactly (integer work: bit-exact)."""
import ctypes
import os
import random
import re

import pytest

from oracle import mapping as om
from paper_2511_02132_b200 import _lib, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "attn_numa.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2511_02132_b200 import build

    build.build()
    return _lib.load()


def test_header_exports_match(lib):
    declared = set(re.findall(r"ATTN_API\s+[\w\s\*]+?\b(attn_\w+)\s*\(", open(HEADER).read()))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), f"{name} not exported"
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (attn_\w+)", out))
    assert declared <= exported


def test_header_flag_values_match_binding():
    """Every mapping flag the binding ORs in has the value the header defines."""
    from paper_2511_02132_b200 import api

    hdr = open(os.path.join(ROOT, "include", "attn_numa.h")).read()
    defs = {m.group(1): int(m.group(2), 16) for m in re.finditer(r"#define ATTN_(\w+) (0x[0-9a-fA-F]+)", hdr)}
    for name in ("ORDER_DESCENDING", "CLUSTER_MULTICAST", "ORDER_ALTERNATE", "SHF_ACC_SHARED", "SHF_ACC_PER_DIE",
                 "BWD_DETERMINISTIC"):
        assert defs[name] == getattr(api, name), name


def test_status_strings_and_version(lib):
    assert lib.attn_status_string(0) == b"ATTN_OK"
    assert lib.attn_status_string(1) == b"ATTN_ERR_INVALID_VALUE"
    assert lib.attn_status_string(2) == b"ATTN_ERR_UNSUPPORTED"
    assert b"sm_100a" in lib.attn_version()


def _fwd(lib, q=1 << 20, k=2 << 20, v=3 << 20, o=4 << 20, B=1, Hq=2, Hkv=2, N=128, d=64, causal=0, scale=0.125,
         mapping=2):
    return lib.attn_fwd(q, k, v, o, B, Hq, Hkv, N, d, causal, scale, mapping)


@pytest.mark.parametrize("kw,status", [
    (dict(q=0), 1), (dict(o=0), 1), (dict(B=0), 1), (dict(N=-1), 1), (dict(Hq=6, Hkv=4), 1),
    (dict(mapping=4), 1), (dict(mapping=-1), 1), (dict(mapping=0x4000), 1), (dict(mapping=0x804), 1), (dict(mapping=0x404), 1), (dict(mapping=0x204), 1), (dict(mapping=0x104), 1), (dict(scale=float("nan")), 1), (dict(scale=float("inf")), 1),
    (dict(d=100), 2), (dict(d=136), 2), (dict(scale=-0.5), 2), (dict(q=(1 << 20) + 8), 2),
    (dict(o=(1 << 20) + 64), 1),   # o overlaps q
])
def test_invalid_arguments_rejected_before_launch(lib, kw, status):
    assert _fwd(lib, **kw) == status
    assert len(lib.attn_last_error()) > 0


def test_non_device_pointers_rejected(lib):
    # plausible arguments but host addresses: never reaches a launch
    buf = (ctypes.c_uint16 * (4 * 2 * 128 * 64))()
    base = ctypes.addressof(buf)
    n = 2 * 128 * 64 * 2
    rc = lib.attn_fwd(base, base + n, base + 2 * n, base + 3 * n, 1, 2, 2, 128, 64, 0, 0.125, 2)
    assert rc != 0


def test_topology_override_validates(lib):
    assert lib.attn_set_topology_override(-1, None, 0, 0) != 0


@pytest.mark.parametrize("mapping", om.MAPPINGS)
def test_schedule_order_matches_oracle(lib, mapping):
    rng = random.Random(7)
    for _ in range(60):
        Hkv = rng.choice([1, 2, 3, 4, 8, 16])
        Hq = Hkv * rng.choice([1, 2, 4])
        B = rng.randint(1, 3)
        N = 128 * rng.randint(1, 12)
        sizes = [rng.randint(60, 80) for _ in range(rng.randint(1, 3))]
        U = (N + 255) // 256
        got = api.attn_schedule_order(B, Hq, Hkv, N, mapping, sizes)
        want = om.build_queues(mapping, B, Hq, Hkv, U, sizes)
        assert got == want, (mapping, B, Hq, Hkv, N, sizes)


@pytest.mark.parametrize("grain", ["shared", "per_die"])
def test_schedule_order_shf_grain_matches_oracle(lib, grain):
    rng = random.Random(29)
    for _ in range(60):
        Hkv = rng.choice([1, 2, 3, 4, 8, 16])
        Hq = Hkv * rng.choice([1, 2, 4])
        B, N = rng.randint(1, 3), 128 * rng.randint(1, 12)
        sizes = [rng.randint(60, 80) for _ in range(rng.randint(1, 3))]
        U = (N + 255) // 256
        got = api.attn_schedule_order(B, Hq, Hkv, N, "swizzled_head_first:" + grain, sizes)
        want = om.build_queues(om.SWIZZLED_HEAD_FIRST, B, Hq, Hkv, U, sizes, shared_acc=grain == "shared")
        assert got == want, (grain, B, Hq, Hkv, N, sizes)
    # the shared grain is the head-first order whatever the die sizes
    got = api.attn_schedule_order(2, 4, 2, 128 * 6, "swizzled_head_first:shared", [2, 1])
    assert got == api.attn_schedule_order(2, 4, 2, 128 * 6, "head_first", [2, 1])


def test_shf_acc_rule_matches_oracle(lib):
    for D in (1, 2, 4):
        for N in (128, 8192, 32768, 64512, 64513, 65536, 98304, 131072, 262144):
            for d in (56, 64, 128):
                for l2 in (0, 50 << 20, 132120576):
                    assert api.attn_shf_acc_shared(D, N, d, l2) == om.shf_acc_shared(D, N, d, l2), (D, N, d, l2)


def test_shf_grain_flags_exclusive(lib):
    fake = [(i + 1) << 20 for i in range(4)]
    rc = lib.attn_fwd(*fake, 1, 2, 2, 128, 64, 0, 0.125, 2 | 0x800 | 0x1000)
    assert rc == 1 and b"exclusive" in lib.attn_last_error()


def test_schedule_order_descending_matches_oracle(lib):
    rng = random.Random(11)
    for _ in range(30):
        Hkv = rng.choice([1, 2, 4, 8])
        Hq = Hkv * rng.choice([1, 2])
        B, N = rng.randint(1, 2), 128 * rng.randint(1, 10)
        U = (N + 255) // 256
        for m in om.MAPPINGS:
            got = api.attn_schedule_order(B, Hq, Hkv, N, m, [74, 74], order="descending")
            assert got == om.descending(om.build_queues(m, B, Hq, Hkv, U, [74, 74]), U)


def test_schedule_order_alternate_matches_oracle(lib):
    rng = random.Random(17)
    for _ in range(30):
        Hkv = rng.choice([1, 2, 3, 4, 8])
        Hq = Hkv * rng.choice([1, 2])
        B, N = rng.randint(1, 2), 128 * rng.randint(1, 10)
        U = (N + 255) // 256
        sizes = [rng.randint(60, 80) for _ in range(rng.randint(1, 3))]
        for m in om.MAPPINGS:
            got = api.attn_schedule_order(B, Hq, Hkv, N, m, sizes, order="alternate")
            assert got == om.alternate(om.build_queues(m, B, Hq, Hkv, U, sizes), U)


def test_schedule_order_cluster_units_match_oracle(lib):
    """ATTN_CLUSTER_MULTICAST: the queues order cluster units exactly as the
    mapping oracle orders units -- head pairs of one KV group (Hq/2 "heads")
    when Hq/Hkv is even, else pairs of adjacent units (ceil(U/2) per head)."""
    rng = random.Random(13)
    for _ in range(40):
        Hkv = rng.choice([1, 2, 3, 4, 8])
        Hq = Hkv * rng.choice([1, 2, 3, 4])
        B, N = rng.randint(1, 2), 128 * rng.randint(1, 12)
        U = (N + 255) // 256
        for m in om.MAPPINGS:
            got = api.attn_schedule_order(B, Hq, Hkv, N, m, [74, 74], cluster=True)
            if (Hq // Hkv) % 2 == 0:
                assert got == om.build_queues(m, B, Hq // 2, Hkv, U, [74, 74])
            else:
                assert got == om.build_queues(m, B, Hq, Hkv, (U + 1) // 2, [74, 74])


def test_backward_rejects_cluster_flag(lib):
    fake = [(i + 1) << 20 for i in range(9)]
    rc = lib.attn_bwd(*fake, 1, 2, 2, 128, 64, 0, 0.125, 2 | 0x200, None)
    assert rc == 2 and b"forward-only" in lib.attn_last_error()


def test_schedule_order_baseline_configs(lib):
    """The BASELINE configs on B200's measured 74/74 split: SHF co-locates every ACC."""
    for (B, Hq, Hkv, N) in ((1, 32, 32, 8192), (1, 128, 128, 32768), (2, 64, 8, 16384)):
        q = api.attn_schedule_order(B, Hq, Hkv, N, "swizzled_head_first", [74, 74])
        assert len(q) == 2 and abs(len(q[0]) - len(q[1])) <= (N // 256) * (Hq // Hkv)
        doms = om.acc_domains(q, Hq, Hkv)
        assert all(len(s) == 1 for s in doms.values())
        assert om.is_bijection(q, B, Hq, N // 256)
