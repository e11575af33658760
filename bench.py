#!/usr/bin/env python
"""Benchmark of the hot path: attention forward TFLOP/s by mapping (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2|C3|C4|C5]
                    [--mapping swizzled_head_first] [--impl ours|reference]

One step = one pass of the whole hot path (topology-aware scheduler + fused
tcgen05 attention kernel: one kernel launch) over one batch of synthetic
bf16 inputs already resident in HBM.  For N > 1 (torchrun, one rank per GPU)
heads are sharded with no data-path collective: the default C2 workload
scales weakly (every rank owns a C2-shaped 32-head shard of a 32N-head
problem); C5 scales strongly (its 128 heads are split over the ranks).
Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 CPU oracle
(oracle/) on a bounded row sample of the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (B, Hq, Hkv, N, d, causal, scaling)        BASELINE.json configs
    "C1": (1, 2, 2, 128, 64, False, "weak"),
    "C2": (1, 32, 32, 8192, 128, False, "weak"),
    "C3": (1, 128, 128, 32768, 128, True, "weak"),
    "C4": (2, 64, 8, 16384, 128, True, "weak"),
    "C5": (1, 128, 128, 131072, 128, True, "strong"),
    # NEXT-2: DeepSeek-V3 prefill (Table 2: MHA 128/128, d = 56; fig:dsmhaperf N 2K-128K)
    "C6": (1, 128, 128, 32768, 56, True, "weak"),
}
METRIC = "attention fwd TFLOP/s (% of bf16 peak) and L2 hit rate by mapping, 1/2/4/8 B200"
MAPS = ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first")


def flops_fwd(B, Hq, N, d, causal, pass_="fwd") -> float:
    """4*B*Hq*N^2*d (two matmuls, eq:fa); the backward counts five matmuls,
    10*B*Hq*N^2*d (eq:ba); causal counts half (FA convention,
    DESIGN.md R14)."""
    f = (10.0 if pass_ == "bwd" else 4.0) * B * Hq * N * N * d
    return f * 0.5 if causal else f


def job_shape(name, world):
    """(B, Hq_total, Hkv_total, N, d, causal, scaling) of the whole job at `world` ranks."""
    B, Hq, Hkv, N, d, causal, scaling = WORKLOADS[name]
    if scaling == "weak":
        Hq, Hkv = Hq * world, Hkv * world
    return B, Hq, Hkv, N, d, causal, scaling


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", 0.0)) or None, "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def load_profile_summary(workload, mapping, cluster=False):
    """ncu --set full summary committed under profiles/ for this workload/mapping, if any."""
    path = os.path.join(ROOT, "profiles", f"ncu_{workload}_{mapping}{'_cluster' if cluster else ''}.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def ncu_fields(prof):
    """Per-mapping ncu evidence (north star: L2 hit rate, tensor-pipe
    utilisation, HBM GB/s) from a committed --set full summary, or None."""
    if not prof:
        return {"l2_hit_rate_pct": None, "tensor_pipe_pct": None, "hbm_gbs": None, "dram_gb_per_launch": None}
    t = prof.get("gpu__time_duration.sum")
    dram = prof.get("dram_bytes_per_launch")
    return {"l2_hit_rate_pct": prof.get("lts__t_sector_hit_rate.pct"),
            "tensor_pipe_pct": prof.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "hbm_gbs": round(dram / t / 1e9, 1) if (dram and t) else None,
            "dram_gb_per_launch": round(dram / 1e9, 3) if dram else None}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML SM clock + throttle reasons sampled in a thread during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.period = [], 0, period_s
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        s = sorted(self.samples)
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(s)}


# ------------------------------------------------------------- our arm (GPU)
def run_ours(a):
    import torch

    from paper_2511_02132_b200 import api, dist as pdist, synth

    rank, world, local = pdist.init()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B, Hq_job, Hkv_job, N, d, causal, scaling = job_shape(a.workload, world)
    shard = pdist.shard_heads(Hq_job, Hkv_job, rank, world)
    hq, hkv = shard.hq, shard.hkv
    scale = 1.0 / math.sqrt(d)
    api.attn_init(local)
    topo = api.attn_topology(local)

    # inputs resident in HBM; rotate over several sets when one set is small
    # enough to survive in L2 between steps (no flush inside the timed region)
    l2 = topo["l2_bytes"]
    set_bytes = 2 * B * (2 * hq + 2 * hkv) * N * d
    n_sets = a.sets if a.sets > 0 else (1 if set_bytes > 4 * l2 else 3)
    sets = []
    for s in range(n_sets):
        q, k, v = synth.make_qkv(B, hq, hkv, N, d, base=s, q_head_offset=shard.q_lo, kv_head_offset=shard.kv_lo,
                                 device=dev)
        sets.append((q, k, v, torch.empty_like(q)))
    l2_note = (f"inputs rotated over {n_sets} sets ({n_sets * set_bytes / 2**20:.0f} MiB > L2 "
               f"{l2 / 2**20:.0f} MiB)" if n_sets > 1 else
               f"one input set of {set_bytes / 2**20:.0f} MiB (L2 {l2 / 2**20:.0f} MiB)")
    l2_note += "; L2 flushed (memset 2xL2) before every step, outside the per-launch events" if a.flush else "; no flush"
    flush_buf = torch.empty(2 * l2, dtype=torch.uint8, device=dev) if a.flush else None
    stream = torch.cuda.current_stream()
    flops_rank = flops_fwd(B, hq, N, d, causal, a.pass_)
    flops_job = flops_fwd(B, Hq_job, N, d, causal, a.pass_)
    bwd_inputs = []
    if a.pass_ == "bwd":  # forward once (untimed) for O and the row LSE; dO seeded like Q
        for s_, (q, k, v, o) in enumerate(sets):
            o2, lse = api.attn_fwd_lse(q, k, v, causal=causal, scale=scale)
            do = synth.make_tensor("q", B, hq, N, d, base=100 + s_, head_offset=shard.q_lo, device=dev)
            bwd_inputs.append((o2, lse, do))

    def step(i, mapping):
        q, k, v, o = sets[i % n_sets]
        if a.pass_ == "bwd":
            o2, lse, do = bwd_inputs[i % n_sets]
            api.attn_bwd(q, k, v, o2, do, lse, causal=causal, scale=scale, mapping=mapping, stream=stream)
        else:
            api.attn_fwd(q, k, v, o, causal=causal, scale=scale, mapping=mapping, stream=stream,
                         cluster=bool(cluster_on[0]))

    cluster_on = [a.cluster if a.pass_ == "fwd" else 0]

    def timed(mapping, steps, warmup, sampler=None):
        for i in range(warmup):
            step(i, mapping)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches = 0
        ctx = sampler if sampler is not None else _Null()
        with ctx:
            e0.record(stream)
            for i in range(steps):
                if flush_buf is not None:
                    flush_buf.zero_()
                evs[i][0].record(stream)
                step(i, mapping)
                evs[i][1].record(stream)
                launches += api.attn_last_launch_info()["kernel_launches"]
            e1.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ms_step = e0.elapsed_time(e1) / steps
        ms_kernel = sum(s.elapsed_time(t) for s, t in evs) / steps
        return pdist.max_over_ranks(ms_step, dev), pdist.max_over_ranks(ms_kernel, dev), launches

    sampler = ClockSampler(local)
    ms_step, ms_kernel, launches = timed(a.mapping, a.steps, a.warmup, sampler)
    clocks = sampler.summary()
    value = flops_job / (ms_step * 1e-3) / 1e12

    # the same workload under the other mappings (fewer steps); forward: each
    # mapping also with the other cluster setting
    by_mapping = {}
    for m in MAPS:
        if m == a.mapping:
            msm = ms_step
        else:
            msm, _, _ = timed(m, max(3, a.steps // 4), 2)
        prof = load_profile_summary(a.workload, m, bool(a.cluster)) if a.pass_ == "fwd" else None
        by_mapping[m] = {"tflops": round(flops_job / (msm * 1e-3) / 1e12, 1), "ms_per_step": round(msm, 4),
                         **(ncu_fields(prof) if a.pass_ == "fwd" else {})}
        if a.pass_ == "fwd":
            cluster_on[0] = 1 - a.cluster
            msc, _, _ = timed(m, max(3, a.steps // 4), 2)
            cluster_on[0] = a.cluster
            profc = load_profile_summary(a.workload, m, not a.cluster)
            by_mapping[m]["cluster" if not a.cluster else "no_cluster"] = {
                "tflops": round(flops_job / (msc * 1e-3) / 1e12, 1), "ms_per_step": round(msc, 4),
                **ncu_fields(profc)}

    # replicated output (N > 1, forward): the kernel epilogue storing O into
    # every rank's buffer over NVLink (attn_fwd_replicated + CUDA IPC) vs the
    # forward followed by an NCCL all-gather of O; device-timed, max over ranks
    replicated = None
    if world > 1 and a.pass_ == "fwd" and not a.no_replicated:
        try:
            replicated = measure_replicated(api, pdist, sets[0], shard, (B, Hq_job, N, d), causal, scale, a.mapping,
                                            rank, world, dev, stream)
        except Exception as e:  # reported, never fatal to the main line
            replicated = {"error": repr(e)[:300]}

    # end to end through the public API on pinned host buffers
    e2e_steps = max(2, min(a.steps, 10))
    if a.pass_ == "fwd":
        qh, kh, vh, _ = sets[0]
        qh, kh, vh = (t.cpu().pin_memory() for t in (qh, kh, vh))
        oh = torch.empty_like(qh).pin_memory()

        def e2e_step():
            api.attn_fwd_host(qh, kh, vh, oh, causal=causal, scale=scale, mapping=a.mapping, stream=stream,
                              cluster=bool(a.cluster))
        h2d = sum(t.numel() * t.element_size() for t in (qh, kh, vh))
        d2h = oh.numel() * oh.element_size()
        e2e_api = "attn_fwd_host (pinned host buffers, H2D + kernel + D2H + sync)"
    else:
        # q, k, v, O, dO, lse host -> device; attn_bwd; dq, dk, dv device -> host
        ins_h = [t.cpu().pin_memory() for t in (*sets[0][:3], *bwd_inputs[0])]
        outs_h = [torch.empty_like(ins_h[i]).pin_memory() for i in range(3)]

        def e2e_step():
            qh_, kh_, vh_, oh_, lseh_, doh_ = ins_h
            api.attn_bwd_host(qh_, kh_, vh_, oh_, doh_, lseh_, *outs_h, causal=causal, scale=scale,
                              mapping=a.mapping, stream=stream)
        h2d = sum(t.numel() * t.element_size() for t in ins_h)
        d2h = sum(t.numel() * t.element_size() for t in outs_h)
        e2e_api = "attn_bwd_host (pinned host q,k,v,O,dO,lse; chunked H2D || kernels || D2H of dq,dk,dv; sync)"
    for _ in range(2):
        e2e_step()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    t_e2e = pdist.max_over_ranks((time.perf_counter() - t0) / e2e_steps, dev)

    peak, peak_sus, peak_src = load_peaks()
    achieved = flops_rank / (ms_kernel * 1e-3) / 1e12
    prof = load_profile_summary(a.workload, a.mapping, bool(a.cluster)) if a.pass_ == "fwd" else None
    traffic = None
    if prof and prof.get("dram_bytes_per_launch") is not None:
        traffic = prof["dram_bytes_per_launch"]
    out = {
        "metric": METRIC if a.pass_ == "fwd" else METRIC.replace("attention fwd", "attention bwd"),
        "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (i.i.d. N(0,1) rounded to bf16, seeded per head)",
        "config": {"workload": a.workload, "B": B, "Hq": Hq_job, "Hkv": Hkv_job, "N": N, "d": d, "causal": causal,
                   "mapping": a.mapping, "pass": a.pass_, "heads_per_gpu": hq,
                   "cluster_multicast": bool(a.cluster) and a.pass_ == "fwd",
                   "parallelism": f"heads sharded over {world} GPU(s), no data-path collective",
                   "l2": l2_note, "flop_convention": ("4*B*Hq*N^2*d, causal x0.5" if a.pass_ == "fwd" else
                                                      "10*B*Hq*N^2*d (5 matmuls), causal x0.5")},
        "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": f"bf16_tflops {peak_src} (burst: one kernel per step)",
                     "kernel_ms": round(ms_kernel, 4)},
        "by_mapping": by_mapping,
        "topology": {"n_domains": topo["n_domains"], "sms_per_domain": topo["sms_per_domain"],
                     "source": topo["source"], "lat_near_cyc": round(topo["lat_near_cyc"], 1),
                     "lat_far_cyc": round(topo["lat_far_cyc"], 1)},
        "e2e": {"value": round(flops_job / t_e2e / 1e12, 2), "unit": "TFLOP/s", "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": d2h * world, "ms_per_step": round(t_e2e * 1e3, 3),
                "api": e2e_api},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if replicated is not None:
        out["replicated_output"] = replicated
    if rank == 0 and world == 1 and not a.no_cpu_baseline and a.pass_ == "fwd":
        out["cpu_baseline"] = cpu_baseline(a.workload, a.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def measure_replicated(api, pdist, qkvo, shard, full_shape, causal, scale, mapping, rank, world, dev, stream,
                       reps=5):
    import torch
    import torch.distributed as tdist

    q, k, v, o = qkvo

    def agree(ok):
        # every rank learns whether all ranks succeeded, so a failure on one
        # rank never leaves the others waiting in a collective below
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MIN)
        return bool(t.item())

    po, err = None, None
    try:
        po = pdist.PeerOutput(full_shape, rank, world, dev)
    except Exception as e:  # noqa: BLE001
        err = repr(e)[:300]
    if not agree(err is None):
        if po is not None:
            po.close()
        return {"error": err or "PeerOutput failed on another rank"}
    dsts = [po.ptrs[rank]] + [p for r, p in enumerate(po.ptrs) if r != rank]
    nccl = tdist.get_backend() == "nccl"
    gbuf = torch.empty((world,) + tuple(o.shape), dtype=o.dtype, device=dev) if nccl else None

    def fused():
        api.attn_fwd_replicated(q, k, v, dsts, full_shape[1], shard.q_lo, causal=causal, scale=scale,
                                mapping=mapping, stream=stream)

    try:  # one checked call before the timed ones
        fused()
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        err = repr(e)[:300]
    if not agree(err is None):
        po.close()
        return {"error": err or "attn_fwd_replicated failed on another rank"}

    def gathered():
        api.attn_fwd(q, k, v, o, causal=causal, scale=scale, mapping=mapping, stream=stream)
        tdist.all_gather_into_tensor(gbuf, o)

    def time_it(fn):
        ts = []
        for i in range(reps + 2):
            torch.cuda.synchronize()
            tdist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        return pdist.max_over_ranks(ts[len(ts) // 2], dev)

    res = {"fused_peer_store_ms": round(time_it(fused), 4),
           "fwd_then_nccl_allgather_ms": round(time_it(gathered), 4) if nccl else None,
           "o_bytes_per_rank": o.numel() * o.element_size(),
           "method": "attn_fwd_replicated: epilogue stores each O tile into all ranks' buffers (CUDA IPC, NVLink "
                     "P2P); vs attn_fwd + all_gather_into_tensor; median of 5, device events, max over ranks"}
    # the fused result must equal the gathered one (heads are independent)
    tdist.barrier()
    if nccl:
        ref = gbuf.permute(1, 0, 2, 3, 4).reshape(full_shape)
        res["bit_identical"] = bool(torch.equal(po.local.view(torch.int16), ref.view(torch.int16)))
    po.close()
    return res


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ----------------------------------------------------------- oracle (CPU)
def _oracle_inputs(name):
    import torch

    from paper_2511_02132_b200 import synth

    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cpu",
                             dtype=torch.float32 if name == "C1" else torch.bfloat16)
    return (B, Hq, Hkv, N, d, causal), (q, k, v)


def _rows(shape, n, seed):
    import numpy as np

    B, Hq, _, N, _, _ = shape
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, B, n), rng.integers(0, Hq, n), rng.integers(0, N, n)], 1).astype(np.int64)


def _row_flops(shape, rows):
    _, _, _, N, d, causal = shape
    keys = (rows[:, 2] + 1) if causal else N
    return float((4.0 * d * keys).sum()) if causal else 4.0 * d * N * len(rows)


def cpu_baseline(name, seconds):
    """The oracle as it stands, on this host's cores, over a bounded row sample."""
    from oracle import attn as oa

    shape, (q, k, v) = _oracle_inputs(name)
    threads = len(os.sched_getaffinity(0))
    oa.set_threads(threads)
    d = shape[4]
    scale = 1.0 / math.sqrt(d)
    probe = _rows(shape, 32, 1)
    t0 = time.perf_counter()
    oa.attention_rows(q, k, v, probe, causal=shape[5], scale=scale)
    per_row = (time.perf_counter() - t0) / len(probe)
    n = int(max(32, min(200000, seconds / max(per_row, 1e-9))))
    rows = _rows(shape, n, 2)
    t0 = time.perf_counter()
    oa.attention_rows(q, k, v, rows, causal=shape[5], scale=scale)
    dt = time.perf_counter() - t0
    fl = _row_flops(shape, rows)
    return {"value": round(fl / dt / 1e12, 6), "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
            "sample": f"{n} random query rows of {name} (fp64 two-pass softmax, {fl / 1e9:.1f} GFLOP) in {dt:.1f} s",
            "seconds": round(dt, 2)}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle
    from oracle import attn as oa

    shape, (q, k, v) = _oracle_inputs(a.workload)
    threads = len(os.sched_getaffinity(0))
    oa.set_threads(threads)
    scale = 1.0 / math.sqrt(shape[4])
    probe = _rows(shape, 16, 1)
    t0 = time.perf_counter()
    oa.attention_rows(q, k, v, probe, causal=shape[5], scale=scale)
    per_row = (time.perf_counter() - t0) / len(probe)
    budget = max(0.05, min(2.0, 90.0 / max(1, a.steps + a.warmup)))  # whole run within ~1.5 min
    n = int(max(8, budget / max(per_row, 1e-9)))
    for i in range(a.warmup):
        oa.attention_rows(q, k, v, _rows(shape, n, 100 + i), causal=shape[5], scale=scale)
    tot_t, tot_f = 0.0, 0.0
    for i in range(a.steps):
        rows = _rows(shape, n, 1000 + i)
        t0 = time.perf_counter()
        oa.attention_rows(q, k, v, rows, causal=shape[5], scale=scale)
        tot_t += time.perf_counter() - t0
        tot_f += _row_flops(shape, rows)
    value = tot_f / tot_t / 1e12
    B, Hq, Hkv, N, d, causal, scaling = job_shape(a.workload, world)
    sample = f"{n} random query rows of {a.workload} per step (fp64 two-pass softmax oracle)"
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(tot_t / a.steps * 1e3, 3),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (i.i.d. N(0,1) rounded to bf16, seeded per head)",
        "config": {"workload": a.workload, "B": B, "Hq": Hq, "Hkv": Hkv, "N": N, "d": d, "causal": causal,
                   "mapping": a.mapping, "parallelism": "CPU oracle on rank 0 host cores"},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--mapping", default="swizzled_head_first", choices=MAPS)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-replicated", action="store_true",
                    help="N > 1: skip the replicated-output (fused peer-store vs NCCL all-gather) measurement")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sets", type=int, default=0, help="resident input sets rotated per step (0: auto)")
    ap.add_argument("--flush", action="store_true", help="memset a 2xL2 buffer before every step")
    ap.add_argument("--cluster", type=int, default=0, choices=(0, 1),
                    help="forward as CTA-pair clusters with K/V multicast (ATTN_CLUSTER_MULTICAST, NEXT-4)")
    ap.add_argument("--pass", dest="pass_", default="fwd", choices=("fwd", "bwd"),
                    help="time the forward (default, the headline) or the backward (NEXT-3)")
    a = ap.parse_args()
    if a.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
