"""Plain-Python reference of the paper's grid-to-die mapping orders.

TEST INFRASTRUCTURE ONLY (never imported by the product package).  Every
function follows the paper's definitions in its own order and notation; the
only library primitives are integer arithmetic and lists.

Paper passages (PAPER.md line numbers, "P:n"; SPEC.md lines "S:n"):
  P:286        grid = batch * num_q_heads * (seqlen_q / BLOCK_M)
  P:100        chunked round-robin dispatch of work-groups to dies, chunk = 1
  P:113-140    fig:wg-swizzle, swizzle_chiplet (the `%` lost in LaTeX, R7)
  P:206, :220  Attention Compute Cluster (ACC): one head (MHA) / group (GQA)
  P:226        Naive Block-first: all heads of block 0, then block 1, ...
  P:246        Naive Head-first: all blocks of head 0, then head 1, ...
  P:236-243    Swizzled Block-first (AITER): block-first order with GQA groups
               pinned to XCDs; keeps locality only when #groups == #XCDs
  S:172        SwizzledBlockFirst: groups with kv_group mod X == x go to XCD x,
               enumerated block-major within the XCD's queue
  P:259-304    Swizzled Head-first: each head's blocks on one die; each die
               serves one ACC at a time; fig:head-first-code (Fig. 7)
  S:55         kv_group = q_head // (H_Q / H_K)
  S:109        batch is the outermost loop (Fig. 7's batch_offset)

B200 readings:
  R6  Fig. 7 listing reconstructed with `%` restored and batch outermost
      (the literal `wid // BATCH` at P:290 is not a bijection for BATCH > 1).
  R8  Per-die queues: within each batch item the ACCs are cut into D
      contiguous ranges proportional to the SMs of each die (Fig. 7 gives
      hpx = H / X equal heads per XCD; equal dies reduce to exactly that).
      If a batch item has fewer ACCs than dies, the cut is taken over the
      global (b, ACC) list; if the whole problem has fewer ACCs than dies,
      the head-major tile list is cut at tile granularity.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

Tile = Tuple[int, int, int]  # (b, h, blk)

BLOCK_FIRST = "block_first"
HEAD_FIRST = "head_first"
SWIZZLED_HEAD_FIRST = "swizzled_head_first"
SWIZZLED_BLOCK_FIRST = "swizzled_block_first"
MAPPINGS = (BLOCK_FIRST, HEAD_FIRST, SWIZZLED_HEAD_FIRST, SWIZZLED_BLOCK_FIRST)


# ---------------------------------------------------------------- attn-grid
def blocks_per_head(N: int, block_m: int) -> int:
    """Fig. 7: blocks_per_head = (SEQLEN_Q + BLOCK_M - 1) // BLOCK_M."""
    return (N + block_m - 1) // block_m


def grid_size(B: int, Hq: int, N: int, block_m: int) -> int:
    """batch * num_q_heads * (seqlen_q / BLOCK_M), ceil for partial blocks."""
    return B * Hq * blocks_per_head(N, block_m)


def validate(B: int, Hq: int, Hkv: int, N: int, block_m: int) -> dict:
    """positive sizes, Hq % Hkv == 0, block_m <= N."""
    if min(B, Hq, Hkv, N, block_m) <= 0:
        raise ValueError("sizes must be positive")
    if Hq % Hkv != 0:
        raise ValueError("non-uniform GQA groups (Hq % Hkv != 0)")
    if block_m > N:
        raise ValueError("block_m exceeds seqlen")
    return {"blocks_per_head": blocks_per_head(N, block_m), "group_size": Hq // Hkv,
            "kind": "MHA" if Hq == Hkv else "GQA"}


def acc_of(Hq: int, Hkv: int, b: int, h: int) -> Tuple[int, int]:
    """P:220 / S:55: ACC = (batch, kv_group), kv_group = h // (Hq/Hkv)."""
    return (b, h // (Hq // Hkv))


# ---------------------------------------------- MI300X formulas (paper's own)
def hardware_dispatch(wgid: int, num_xcd: int, chunk: int = 1) -> int:
    """chunked round-robin work-group -> XCD."""
    return (wgid // chunk) % num_xcd


def swizzle_chiplet(wgid: int, grid: int, num_xcd: int) -> int:
    """fig:wg-swizzle with `xcd = wgid % NUM_XCD` restored (R7)."""
    wgids_per_xcd = grid // num_xcd
    xcd = wgid % num_xcd
    local_wgid = wgid // num_xcd
    return xcd * wgids_per_xcd + local_wgid


def map_tile_mi300(strategy: str, wid: int, B: int, H: int, nblk: int, X: int) -> Tile:
    """SPEC map_tile: linear work-group id -> (b, h, blk), batch outermost."""
    per_batch = H * nblk
    b, w = wid // per_batch, wid % per_batch
    if strategy == BLOCK_FIRST:
        return (b, w % H, w // H)
    if strategy == HEAD_FIRST:
        return (b, w // nblk, w % nblk)
    if strategy == SWIZZLED_HEAD_FIRST:
        hpx = H // X
        x, kk = w % X, w // X
        return (b, x * hpx + kk // nblk, kk % nblk)
    raise ValueError(strategy)


def fig7_swizzled_head_first(wid: int, BATCH: int, H: int, nblk: int, X: int) -> Tile:
    """fig:head-first-code reconstructed with `%` restored (R6).

      w      = wid % (H * B)             # B = blocks_per_head
      head   = (w % X) * hpx + w // (X * B)
      block  = (w % (X * B)) // X
      batch  = (wid // (B * H)) % BATCH
    """
    Bk = nblk
    hpx = H // X
    w = wid % (H * Bk)
    head = (w % X) * hpx + w // (X * Bk)
    block = (w % (X * Bk)) // X
    batch = (wid // (Bk * H)) % BATCH
    return (batch, head, block)


# ------------------------------------------------------ B200 per-die queues
def _prop_cuts(total: int, sizes: Sequence[int]) -> List[int]:
    """Cut [0,total) into len(sizes) contiguous ranges proportional to sizes
    (rounded to nearest): cut_d = (total * sum_{e<d} S_e + S/2) // S."""
    S = sum(sizes)
    cuts, acc = [], 0
    for s in sizes:
        cuts.append((total * acc + S // 2) // S)
        acc += s
    cuts.append(total)
    return cuts


def head_major_tiles(B: int, Hq: int, nblk: int) -> List[Tile]:
    """P:246 order: for b, for h, for blk (batch outermost)."""
    return [(b, h, k) for b in range(B) for h in range(Hq) for k in range(nblk)]


def block_major_tiles(B: int, Hq: int, nblk: int) -> List[Tile]:
    """P:226 order: for b, for blk, for h."""
    return [(b, h, k) for b in range(B) for k in range(nblk) for h in range(Hq)]


def shf_acc_shared(n_domains: int, N: int, d: int, l2_bytes: int) -> bool:
    """R23 (B200 reading of P:259-270): the dies share one L2, so swizzled
    head-first keeps n_domains ACC footprints (K and V of one KV head:
    2 tensors x N x d x 2 bytes each) live in it at once; when together they
    exceed half of the L2, each ACC is shared by all dies instead."""
    footprint_one_acc = 2 * N * d * 2
    return n_domains > 1 and l2_bytes > 0 and n_domains * footprint_one_acc > l2_bytes // 2


def build_queues(mapping: str, B: int, Hq: int, Hkv: int, nblk: int,
                 domain_sizes: Sequence[int], shared_acc: bool = False) -> List[List[Tile]]:
    """Ordered work queues a B200 persistent grid pops from.

    block_first / head_first: one queue shared by every SM of every die
    (the B200 analogue of round-robin dispatch: consecutive tiles of a head
    land on SMs of both dies).  swizzled_head_first: one queue per die
    (R8), each die serving its ACCs one at a time in head-major order; with
    shared_acc (R23) all dies serve the same ACC: they form one capacity
    domain, and swizzled head-first over one domain is head-first (S:189,
    S:206).
    """
    if mapping == BLOCK_FIRST:
        return [block_major_tiles(B, Hq, nblk)]
    if mapping == HEAD_FIRST:
        return [head_major_tiles(B, Hq, nblk)]
    D = len(domain_sizes)
    G = Hq // Hkv
    if mapping == SWIZZLED_BLOCK_FIRST:
        # S:172 / P:243: die d serves the KV groups g with g mod D == d, block-major
        # within its queue (for b: for blk: for its groups' heads).  With one die
        # this is plain block-first.
        if D == 1:
            return [block_major_tiles(B, Hq, nblk)]
        queues = [[] for _ in range(D)]
        for d in range(D):
            groups = [g for g in range(Hkv) if g % D == d]
            for b in range(B):
                for k in range(nblk):
                    for g in groups:
                        queues[d].extend((b, h, k) for h in range(g * G, (g + 1) * G))
        return queues
    if mapping != SWIZZLED_HEAD_FIRST:
        raise ValueError(mapping)
    if D == 1:
        return [head_major_tiles(B, Hq, nblk)]
    queues: List[List[Tile]] = [[] for _ in range(D)]
    if shared_acc:
        return [head_major_tiles(B, Hq, nblk)]
    if Hkv >= D:
        # Fig. 7 generalised: per batch item, ACCs [cut_d, cut_{d+1}) -> die d.
        cuts = _prop_cuts(Hkv, domain_sizes)
        for b in range(B):
            for d in range(D):
                for g in range(cuts[d], cuts[d + 1]):
                    for h in range(g * G, (g + 1) * G):
                        queues[d].extend((b, h, k) for k in range(nblk))
        return queues
    if B * Hkv >= D:
        # fewer ACCs per batch item than dies: cut the global (b, ACC) list.
        accs = [(b, g) for b in range(B) for g in range(Hkv)]
        cuts = _prop_cuts(len(accs), domain_sizes)
        for d in range(D):
            for (b, g) in accs[cuts[d]:cuts[d + 1]]:
                for h in range(g * G, (g + 1) * G):
                    queues[d].extend((b, h, k) for k in range(nblk))
        return queues
    # fewer ACCs than dies overall: split the head-major list at tile granularity.
    tiles = head_major_tiles(B, Hq, nblk)
    cuts = _prop_cuts(len(tiles), domain_sizes)
    return [tiles[cuts[d]:cuts[d + 1]] for d in range(D)]


def descending(queues: List[List[Tile]], nblk: int) -> List[List[Tile]]:
    """The same queues with every (b, h)'s blocks visited last-first (DESIGN.md
    R19: an order knob applied identically under every mapping)."""
    return [[(b, h, nblk - 1 - k) for (b, h, k) in q] for q in queues]


def alternate(queues: List[List[Tile]], nblk: int) -> List[List[Tile]]:
    """The same queues with queue d's (b, h) blocks visited last-first when d
    is odd (R22; a schedule knob, never part of the result)."""
    return [q if d % 2 == 0 else [(b, h, nblk - 1 - k) for (b, h, k) in q] for d, q in enumerate(queues)]


def is_bijection(queues: List[List[Tile]], B: int, Hq: int, nblk: int) -> bool:
    """every tile appears exactly once across the queues."""
    flat = [t for q in queues for t in q]
    return len(flat) == B * Hq * nblk and set(flat) == set(head_major_tiles(B, Hq, nblk))


def acc_domains(queues: List[List[Tile]], Hq: int, Hkv: int) -> dict:
    """ACC -> set of queue (die) indices that hold any of its tiles."""
    out: dict = {}
    for d, q in enumerate(queues):
        for (b, h, _k) in q:
            out.setdefault(acc_of(Hq, Hkv, b, h), set()).add(d)
    return out
