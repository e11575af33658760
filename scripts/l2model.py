"""Analytic L2 model of the K/V reuse each mapping delivers (NEXT-4, second half).

Predicts, for a workload x mapping, the L2 hit rate of the K/V stream and the
DRAM bytes per launch, to be set against the ncu captures in profiles/.  It
is the SPEC's cache-simulation idea re-derived for B200 and fed
with B200 facts measured by this repo:

* schedule: the library's own host queue builder (attn_schedule_order, the
  exact (b, h, unit) order the on-device scheduler pops), per-die queues for
  the swizzled mappings with tail stealing, one shared queue otherwise;
* execution: the persistent grid's 148 CTAs (74 CTA pairs with cluster
  multicast) stream their unit's 128-key blocks (K and V tile) at one block
  per tick times a per-unit speed in [1 - spread, 1 + spread] (CTAs drift
  apart on the GPU: causal diagonal blocks, wake latencies, clocks); a CTA
  pops its next unit as soon as it finishes one (dynamic scheduler).  The
  spread is the model's one calibrated parameter (fit on C3 head-first);
* cache: ONE unified LRU of the L2 size -- the topology probe found B200's L2
  to be a single address-hashed pool with no near-die replication of far
  lines, so die locality does not enter;
* traffic: K/V blocks are read through the LRU; each unit's Q (evict-first
  policy) always misses and never occupies the cache; O is written once and
  occupies the LRU like any line.

Not an oracle: analysis tooling only (it never touches the GPU and is not on
the product path).  Usage: python scripts/l2model.py [C2,C3,C4] [--cluster].
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

BLOCK = 128          # keys per K/V block and rows per query block (kernel constants)
UNIT_ROWS = 256      # rows per work unit (two query blocks)
SPREAD = 0.0         # calibrated per-unit speed spread (NEXT-4 model)


class _LRU:
    def __init__(self, cap):
        self.cap, self.d = cap, collections.OrderedDict()

    def access(self, key) -> bool:
        if key in self.d:
            self.d.move_to_end(key)
            return True
        self.d[key] = None
        if len(self.d) > self.cap:
            self.d.popitem(last=False)
        return False


class _Random:
    """Random replacement (seeded): a miss evicts a uniformly chosen line."""

    def __init__(self, cap, seed):
        import random
        self.cap, self.slot_of, self.keys, self.rng = cap, {}, [], random.Random(seed)

    def access(self, key) -> bool:
        if key in self.slot_of:
            return True
        if len(self.keys) < self.cap:
            self.slot_of[key] = len(self.keys)
            self.keys.append(key)
        else:
            i = self.rng.randrange(self.cap)
            del self.slot_of[self.keys[i]]
            self.keys[i] = key
            self.slot_of[key] = i
        return False


def unit_kv_blocks(u: int, nblk: int, causal: bool) -> int:
    """Key blocks unit u (query blocks 2u, 2u+1) streams -- attn_fwd_sm100.cuh unit_blocks."""
    has1 = 2 * u + 1 < nblk
    if causal:
        return 2 * u + 2 if has1 else 2 * u + 1
    return nblk


def _schedule(B, Hq, Hkv, N, mapping, sms_per_domain, order, cluster):
    from paper_2511_02132_b200 import api  # host-side queue builder (no GPU needed)
    return api.attn_schedule_order(B, Hq, Hkv, N, mapping, sms_per_domain, order=order, cluster=cluster)


def simulate(B: int, Hq: int, Hkv: int, N: int, d: int, causal: bool, mapping: str,
             sms_per_domain=(74, 74), l2_bytes: int = 126 * 2**20, order: str = "ascending",
             cluster: bool = False, queues=None, spread: float = 0.0, policy: str = "lru",
             seed: int = 1) -> dict:
    """Tick simulation of the grid against an LRU L2; returns hit rates and
    DRAM bytes per launch.  spread = 0 is exact lockstep."""
    G = Hq // Hkv
    nblk = (N + BLOCK - 1) // BLOCK
    U = (N + UNIT_ROWS - 1) // UNIT_ROWS
    pair_heads = cluster and G % 2 == 0
    if queues is None:
        queues = _schedule(B, Hq, Hkv, N, mapping, list(sms_per_domain), order, cluster)
    blk_bytes = 2 * BLOCK * d * 2            # K and V tiles of one key block (bf16)
    tile_bytes = BLOCK * d * 2
    cap = max(1, l2_bytes // blk_bytes)      # LRU capacity in K/V-block entries (O lines count alike)

    # workers: one per SM (per CTA pair with clusters), grouped by die
    per_dom = [s // (2 if cluster else 1) for s in sms_per_domain]
    worker_dom = [dm for dm, n in enumerate(per_dom) for _ in range(n)]
    nq = len(queues)
    pos = [0] * nq

    def pop(dom: int):
        q0 = dom if nq > 1 else 0
        for t in range(nq):
            qi = (q0 + t) % nq
            if pos[qi] < len(queues[qi]):
                e = queues[qi][pos[qi]]
                pos[qi] += 1
                return e
        return None

    def work_of(e):
        """(kv head index, #blocks streamed, rows of output) of a scheduler entry."""
        b, h, u = e
        if not cluster:
            return b * Hkv + h // G, unit_kv_blocks(u, nblk, causal), min(UNIT_ROWS, N - u * UNIT_ROWS)
        if pair_heads:   # unit u of heads 2h, 2h+1 (one KV group)
            rows = min(UNIT_ROWS, N - u * UNIT_ROWS)
            return b * Hkv + (2 * h) // G, unit_kv_blocks(u, nblk, causal), 2 * rows
        u0, u1 = 2 * u, 2 * u + 1   # adjacent units of head h
        n = unit_kv_blocks(u0, nblk, causal)
        rows = min(UNIT_ROWS, N - u0 * UNIT_ROWS)
        if u1 < U:
            n = max(n, unit_kv_blocks(u1, nblk, causal))
            rows += min(UNIT_ROWS, N - u1 * UNIT_ROWS)
        return b * Hkv + h // G, n, rows

    if policy == "lru":
        cache = _LRU(cap)
    elif policy == "random":
        cache = _Random(cap, seed)
    else:
        raise ValueError("policy must be 'lru' or 'random'")
    kv_hit = kv_miss = 0
    q_bytes = o_bytes = 0
    o_seq = 0
    n_units = [0]

    def speed() -> float:
        # low-discrepancy spread of per-unit speeds (deterministic)
        n_units[0] += 1
        frac = (n_units[0] * 0.6180339887498949) % 1.0
        return 1.0 + spread * (2.0 * frac - 1.0)

    state = []   # per worker: [kvh, next block, n blocks, rows, progress, speed] or None
    for w in range(len(worker_dom)):
        e = pop(worker_dom[w])
        if e is None:
            state.append(None)
        else:
            kvh, n, rows = work_of(e)
            state.append([kvh, 0, n, rows, 0.0, speed()])
            q_bytes += rows * d * 2
    active = sum(s is not None for s in state)
    while active:
        for w, s in enumerate(state):
            if s is None:
                continue
            kvh, j, n, rows, prog, sp = s
            prog += sp
            while j < n and j < prog:
                if cache.access((kvh, j)):
                    kv_hit += 1
                else:
                    kv_miss += 1
                j += 1
            s[1], s[4] = j, prog
            if j >= n:   # unit done: O written, next unit
                o_bytes += rows * d * 2
                nlines = max(1, (rows * d * 2) // blk_bytes)
                for _ in range(nlines):
                    cache.access(("o", o_seq))
                    o_seq += 1
                e = pop(worker_dom[w])
                if e is None:
                    state[w] = None
                    active -= 1
                else:
                    kvh2, n2, rows2 = work_of(e)
                    state[w] = [kvh2, 0, n2, rows2, 0.0, speed()]
                    q_bytes += rows2 * d * 2
    kv_bytes = (kv_hit + kv_miss) * blk_bytes
    dram = kv_miss * blk_bytes + q_bytes + o_bytes
    # all-traffic sector hit rate if O writes count as hits and Q reads as misses
    hit_all = (kv_hit * blk_bytes + o_bytes) / max(1, kv_bytes + q_bytes + o_bytes)
    return {"kv_hit_rate_pct": 100.0 * kv_hit / max(1, kv_hit + kv_miss), "hit_rate_all_pct": 100.0 * hit_all,
            "dram_gb": dram / 1e9, "kv_l2_gb": kv_bytes / 1e9, "q_gb": q_bytes / 1e9, "o_gb": o_bytes / 1e9,
            "kv_miss_gb": kv_miss * blk_bytes / 1e9, "l2_entries": cap, "tile_bytes": tile_bytes}


def main():
    from bench import WORKLOADS
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="?", default="C2,C3,C4")
    ap.add_argument("--cluster", action="store_true")
    ap.add_argument("--sms", default="70,78", help="SMs per die (the probe's split)")
    ap.add_argument("--l2-mib", type=float, default=126.0)
    ap.add_argument("--spread", type=float, default=SPREAD, help="per-unit speed spread (calibrated)")
    ap.add_argument("--json", default=None, help="write the table here")
    a = ap.parse_args()
    sms = [int(x) for x in a.sms.split(",")]
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles")
    rows = []
    for name in a.configs.split(","):
        B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
        for m in ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first"):
            r = simulate(B, Hq, Hkv, N, d, causal, m, sms, int(a.l2_mib * 2**20), cluster=a.cluster,
                         spread=a.spread)
            prof = os.path.join(root, f"ncu_{name}_{m}{'_cluster' if a.cluster else ''}.json")
            meas = json.load(open(prof)) if os.path.exists(prof) else {}
            row = {"workload": name, "mapping": m, "cluster": a.cluster, **{k: round(v, 3) for k, v in r.items()},
                   "ncu_hit_rate_pct": meas.get("lts__t_sector_hit_rate.pct"),
                   "ncu_dram_gb": round(meas["dram_bytes_per_launch"] / 1e9, 3) if meas else None}
            rows.append(row)
            print(f"{name} {m:22s} model: K/V hit {r['kv_hit_rate_pct']:5.1f}%  all {r['hit_rate_all_pct']:5.1f}%  "
                  f"DRAM {r['dram_gb']:8.2f} GB | ncu: hit {row['ncu_hit_rate_pct']}  DRAM {row['ncu_dram_gb']} GB",
                  flush=True)
    if a.json:
        json.dump(rows, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
