#!/usr/bin/env python
"""Benchmark of the hot path: attention forward TFLOP/s by mapping (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C1..C6]
                    [--mapping swizzled_head_first] [--cluster 0|1] [--ncu auto|on|off]
                    [--impl ours|reference]

One step = one pass of the whole hot path (topology-aware scheduler + fused
tcgen05 attention kernel: one kernel launch) over one batch of synthetic
bf16 inputs already resident in HBM.  The default workload is BASELINE.json
config 5, the paper's extreme point and the north-star target (MHA 128 heads
x 131072 tokens, causal, d = 128): SHF is timed for
`value`, and block-first, head-first, SHF and swizzled block-first are each
timed plain and as CTA-pair clusters in the same run (`by_mapping`), each
with the L2 hit rate, tensor-pipe utilisation, HBM GB/s, DRAM and cross-die
bytes that an ncu child process measures on one launch per variant IN THIS
RUN (`--ncu`).  For N > 1 (torchrun, one rank per GPU) heads are sharded
with no data-path collective: C5 scales strongly (its 128 heads are split),
the other workloads weakly.  Rank 0 prints ONE JSON line.
`--impl reference` times the fp64 CPU oracle (oracle/) instead, on a bounded
row sample of the same workload (tier framing: the oracle is the reference
arm; there is no reference implementation to install).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import subprocess
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
# swizzled head-first at the paper's literal grain (one die per ACC) beside the
# library's choice (R23: ACCs shared by the dies when the dies' K/V
# footprints overflow the shared L2); reported in by_mapping
VARIANT_MAPS = MAPS + ("swizzled_head_first:per_die",)
# ncu metrics of the per-mapping evidence (north star: L2 hit rate, tensor-pipe
# utilisation, HBM GB/s); R13: sector hit rate over all ops plus the read-only rate
NCU_METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "lts__t_sector_hit_rate.pct", "lts__t_sector_op_read_hit_rate.pct", "lts__t_sectors.sum",
               "lts__t_sectors_srcunit_ltcfabric.sum",
               "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
               "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
               "sm__cycles_elapsed.avg.per_second")


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
    """(burst, sustained, source) bf16 dense TFLOP/s: the driver-measured
    MEASURED_PEAKS.json, else the B200_PROFILING.md fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", 0.0)) or None, "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def mapping_rounds(ms_step: float):
    """by_mapping protocol for a step of ms_step ms: (timed steps per chunk,
    untimed settle steps before each chunk, interleaved rounds).  A chunk is
    ~300 ms of back-to-back steps (at least one), the settle half as long (at
    least one step), and the rounds give ~2 s of timed steps per variant
    (3..50 rounds)."""
    ms = max(ms_step, 1e-3)
    chunk = max(1, int(round(300.0 / ms)))
    settle = max(1, chunk // 2)
    rounds = max(3, min(50, int(round(2000.0 / (chunk * ms)))))
    return chunk, settle, rounds


def variant_key(mapping, cluster, order="ascending"):
    return f"{mapping}{'+cluster' if cluster else ''}{'' if order == 'ascending' else '+' + order}"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML SM clock + throttle reasons sampled in a thread during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.samples, self.power, self.reasons, self.period = [], [], 0, period_s
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

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
        except Exception:
            pass

    def _run(self):
        self._sample()  # at least one sample even for a region shorter than the period
        while not self._stop.wait(self.period):
            self._sample()

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
        out = {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(s),
               "sm_mhz_min": s[0]}
        if self.power:
            out["power_w_median"] = round(sorted(self.power)[len(self.power) // 2], 1)
        return out


# ------------------------------------------------ in-run ncu (per variant)
def ncu_child(a):
    """Run under ncu by ncu_measure(): one attn_fwd launch per variant on the
    parent rank's shard shape (inputs seeded exactly like the parent's)."""
    import torch

    from paper_2511_02132_b200 import api, synth

    torch.cuda.set_device(a.device)
    B, hq, hkv, N, d, causal, q_lo, kv_lo = (int(x) for x in a.ncu_child.split(","))
    q, k, v = synth.make_qkv(B, hq, hkv, N, d, base=0, q_head_offset=q_lo, kv_head_offset=kv_lo,
                             device=f"cuda:{a.device}")
    o = torch.empty_like(q)
    api.attn_init(a.device)
    for spec in a.variants.split(";"):
        m, cl, order = spec.split("/")
        api.attn_fwd(q, k, v, o, causal=bool(causal), scale=1.0 / math.sqrt(d), mapping=m, order=order,
                     cluster=cl == "1")
        torch.cuda.synchronize()


def _ncu_value(v: str, unit: str):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "nsecond": 1e-9,
             "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
             "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1.0,
             "cycle/nsecond": 1e9, "cycle/usecond": 1e6}.get(unit)
    return x * scale if scale is not None else x


def ncu_measure(shape, variants, device: int, timeout_s: float):
    """One ncu process around ncu_child: every attention launch profiled with
    the NCU_METRICS (caches flushed before each launch, clocks unlocked).
    Returns ({variant key: fields}, provenance dict)."""
    ncu = "/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else "ncu"
    log = os.path.join("/tmp", f"attn_bench_ncu_{os.getpid()}.csv")
    spec = ";".join(f"{m}/{int(cl)}/{o}" for (m, cl, o) in variants)
    cmd = [ncu, "--csv", "--print-units", "base", "--log-file", log, "--clock-control", "none",
           "--cache-control", "all", "-k", "regex:attn_fwd_sm100", "--metrics", ",".join(NCU_METRICS),
           sys.executable, os.path.join(ROOT, "bench.py"), "--ncu-child", ",".join(str(int(x)) for x in shape),
           "--variants", spec, "--device", str(device)]
    t0 = time.time()
    prov = {"source": "measured in this run: ncu child process, one launch per variant",
            "command": " ".join(cmd[:13]) + " ... bench.py --ncu-child", "metrics": list(NCU_METRICS)}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, cwd=ROOT)
        prov["rc"] = r.returncode
        if r.returncode != 0:
            prov["error"] = (r.stderr or r.stdout)[-400:]
    except Exception as e:  # noqa: BLE001 -- reported, never fatal
        prov["rc"], prov["error"] = None, repr(e)[:300]
    prov["seconds"] = round(time.time() - t0, 1)
    per = {}
    try:
        text = open(log).read()
        os.unlink(log)
    except OSError:
        text = ""
    lines = text.splitlines()
    start = next((i for i, l in enumerate(lines) if l.startswith('"ID"')), None)
    if start is not None:
        for row in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
            if "attn_fwd_sm100" not in row.get("Kernel Name", ""):
                continue
            per.setdefault(row["ID"], {})[row["Metric Name"]] = _ncu_value(row["Metric Value"], row["Metric Unit"])
    out = {}
    for (m, cl, o), (_, vals) in zip(variants, sorted(per.items(), key=lambda kv: int(kv[0]))):
        t = vals.get("gpu__time_duration.sum")
        rb, wb = vals.get("dram__bytes_read.sum"), vals.get("dram__bytes_write.sum")
        dram = (rb + wb) if rb is not None and wb is not None else None
        fab = vals.get("lts__t_sectors_srcunit_ltcfabric.sum")
        hz = vals.get("sm__cycles_elapsed.avg.per_second")
        out[variant_key(m, cl, o)] = {
            "l2_hit_rate_pct": vals.get("lts__t_sector_hit_rate.pct"),
            "l2_read_hit_rate_pct": vals.get("lts__t_sector_op_read_hit_rate.pct"),
            "tensor_pipe_pct": vals.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "xu_pipe_pct": vals.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),  # MUFU (exp2)
            "hbm_gbs": round(dram / t / 1e9, 1) if dram and t else None,
            "dram_gb_per_launch": round(dram / 1e9, 3) if dram is not None else None,
            "cross_die_gb_per_launch": round(fab * 32 / 1e9, 3) if fab is not None else None,
            "sm_ghz": round(hz / 1e9, 3) if hz else None,
            "ncu_ms": round(t * 1e3, 3) if t else None,
            "dram_bytes": dram,
        }
    prov["kernels_profiled"] = len(per)
    return out, prov


# ------------------------------------------------------------- our arm (GPU)
def run_ours(a):
    import torch

    from paper_2511_02132_b200 import api, dist as pdist, synth

    rank, world, local = pdist.init(nccl_debug_init=True, force=a.replicated)
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
    if n_sets > 1:
        l2_note = f"inputs rotated over {n_sets} sets ({n_sets * set_bytes / 2**20:.0f} MiB > L2 {l2 / 2**20:.0f} MiB)"
    else:
        l2_note = f"inputs larger than L2 ({set_bytes / 2**30:.1f} GiB per step vs L2 {l2 / 2**20:.0f} MiB)"
    l2_note += "; L2 flushed (memset 2xL2) before every step, outside the per-launch events" if a.flush else \
        "; no flush"
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

    def step(i, var):
        mapping, cl, order = var
        q, k, v, o = sets[i % n_sets]
        if a.pass_ == "bwd":
            o2, lse, do = bwd_inputs[i % n_sets]
            api.attn_bwd(q, k, v, o2, do, lse, causal=causal, scale=scale, mapping=mapping, order=order,
                         stream=stream)
        else:
            api.attn_fwd(q, k, v, o, causal=causal, scale=scale, mapping=mapping, order=order, stream=stream,
                         cluster=cl)

    def timed(var, steps, warmup, sampler=None):
        for i in range(warmup):
            step(i, var)
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
                step(i, var)
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

    main_var = (a.mapping, bool(a.cluster) and a.pass_ == "fwd", a.order)
    sampler = ClockSampler(local)
    ms_step, ms_kernel, launches = timed(main_var, a.steps, a.warmup, sampler)
    shf_grain = "shared" if api.attn_last_launch_info().get("shf_acc_shared") else "per_die"
    clocks = sampler.summary()
    value = flops_job / (ms_step * 1e-3) / 1e12

    # every mapping on the same inputs in the same run, plain and (forward) as
    # CTA-pair clusters; fewer steps each
    variants = [(m, cl, "ascending") for m in VARIANT_MAPS for cl in ((False, True) if a.pass_ == "fwd" else (False,))]
    if main_var not in variants:
        variants.append(main_var)
    # Interleaved rounds so every variant sees the same thermal / power-cap
    # state over the run; the value variant's own line above is the contract's
    # timed region.  Under the power cap the SM clock follows the previous
    # kernels' draw with a lag, and a step right after another variant inherits
    # its clock (measured at C3: SHF as clusters 26.5 ms alone, 36-37 ms right
    # after a block-first step), so each round runs a CHUNK of back-to-back
    # steps per variant (~300 ms), the first half untimed (settle), the second
    # half timed as one event pair; by_mapping = median over ~6 rounds of the
    # per-step chunk times (about 2 s timed per variant).
    chunk, settle, rounds = mapping_rounds(ms_step)
    per_var = {v: [] for v in variants}
    for v in variants:  # one untimed step each (descriptors, first-touch)
        step(0, v)
    torch.cuda.synchronize()
    for r in range(rounds):
        for vi, v in enumerate(variants):
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            for i in range(settle):
                step(i + 1, v)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for i in range(chunk):
                step(r * len(variants) + vi + i, v)  # rotate the input sets step by step
            ev1.record(stream)
            torch.cuda.synchronize()
            per_var[v].append(pdist.max_over_ranks(ev0.elapsed_time(ev1) / chunk, dev))
    by_mapping = {}
    for v in variants:
        ts = sorted(per_var[v])
        msm = ts[len(ts) // 2]
        by_mapping[variant_key(*v)] = {"tflops": round(flops_job / (msm * 1e-3) / 1e12, 1),
                                       "ms_per_step": round(msm, 4),
                                       "timing": f"median of {rounds} interleaved rounds of {chunk} timed steps "
                                                 f"after {settle} untimed ones of the same variant"}

    # per-variant ncu evidence measured now, on this rank's shard (rank 0)
    ncu_prov = None
    ncu_on = a.ncu == "on" or (a.ncu == "auto" and a.pass_ == "fwd")
    if ncu_on and rank == 0:
        shape = (B, hq, hkv, N, d, int(causal), shard.q_lo, shard.kv_lo)
        per, ncu_prov = ncu_measure(shape, variants, local, a.ncu_timeout)
        for key, fields in per.items():
            by_mapping.setdefault(key, {}).update({k: v for k, v in fields.items() if k != "dram_bytes"})
    if world > 1:
        torch.distributed.barrier()

    # replicated output (forward): the kernel epilogue storing O into every
    # rank's buffer (attn_fwd_replicated + CUDA IPC) vs the forward followed by
    # an NCCL all-gather of O; device-timed, max over ranks
    replicated = None
    if (world > 1 or a.replicated) and a.pass_ == "fwd" and not a.no_replicated:
        try:
            replicated = measure_replicated(api, pdist, sets[0], shard, (B, Hq_job, N, d), causal, scale,
                                            a.mapping, rank, world, dev, stream)
        except Exception as e:  # reported, never fatal to the main line
            replicated = {"error": repr(e)[:300]}

    # end to end through the public API on pinned host buffers
    e2e_steps = max(2, min(a.steps, 10))
    if a.pass_ == "fwd":
        qh, kh, vh, _ = sets[0]
        qh, kh, vh = (t.cpu().pin_memory() for t in (qh, kh, vh))
        oh = torch.empty_like(qh).pin_memory()

        def e2e_step():
            api.attn_fwd_host(qh, kh, vh, oh, causal=causal, scale=scale, mapping=a.mapping, order=a.order,
                              stream=stream, cluster=main_var[1])
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

    # roofline of the (single) kernel: algorithmic flops per launch / event time
    peak_burst, peak_sus, peak_src = load_peaks()
    timed_s = ms_step * a.steps * 1e-3
    sustained = peak_sus is not None and timed_s >= 1.0
    peak = peak_sus if sustained else peak_burst
    achieved = flops_rank / (ms_kernel * 1e-3) / 1e12
    # exp-unit ceiling: one exp2 per (row, key) for 4d
    # forward flops (10d backward); MUFU.EX2 16 per clock per SM (measured,
    # scripts/micro/mufu_rate.cu) with 1 in 8 exps on the FMA-pipe polynomial
    # (x 8/7), at the maximum SM clock.  Below the tensor peak (d <= 64) the
    # kernel is ALU-bound and the roofline uses it.
    exp_per_clk_sm = 16.0 * 8.0 / 7.0
    flops_per_exp = (10.0 if a.pass_ == "bwd" else 4.0) * d
    max_mhz = clocks.get("sm_max_mhz") or 1965
    exp_ceiling = exp_per_clk_sm * topo["num_sms"] * max_mhz * 1e6 * flops_per_exp / 1e12
    main_ncu = by_mapping.get(variant_key(*main_var), {})
    traffic = None
    if main_ncu.get("dram_gb_per_launch") is not None:
        traffic = round(main_ncu["dram_gb_per_launch"] * 1e9)
    alg_bytes = 2.0 * B * N * d * (2 * hq + 2 * hkv)
    out = {
        "metric": METRIC if a.pass_ == "fwd" else METRIC.replace("attention fwd", "attention bwd"),
        "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (i.i.d. N(0,1) rounded to bf16, seeded per head)",
        "config": {"workload": a.workload, "B": B, "Hq": Hq_job, "Hkv": Hkv_job, "N": N, "d": d, "causal": causal,
                   "mapping": a.mapping, "order": a.order, "pass": a.pass_, "heads_per_gpu": hq,
                   "shf_acc_grain": (shf_grain + " (DESIGN.md R23)") if a.mapping.startswith("swizzled_head_first")
                   else None,
                   "cluster_multicast": main_var[1],
                   "parallelism": f"heads sharded over {world} GPU(s), no data-path collective",
                   "l2": l2_note, "flop_convention": ("4*B*Hq*N^2*d, causal x0.5" if a.pass_ == "fwd" else
                                                      "10*B*Hq*N^2*d (5 matmuls), causal x0.5")},
        "roofline": {"bound": "tensor" if exp_ceiling >= peak else "alu", "achieved": round(achieved, 1),
                     "peak": round(min(peak, exp_ceiling), 1), "unit": "TFLOP/s",
                     "frac": round(achieved / min(peak, exp_ceiling), 4), "traffic": traffic,
                     "tensor_peak": peak,
                     "exp_ceiling": round(exp_ceiling, 1),
                     "exp_ceiling_source": f"16 MUFU.EX2/clk/SM x 8/7 (1/8 polynomial) x {topo['num_sms']} SMs x "
                                           f"{max_mhz} MHz x {flops_per_exp:.0f} flop per exp",
                     "peak_source": ("exp_ceiling (the exps bound this head dim, DESIGN.md section 6)"
                                     if exp_ceiling < peak else
                                     f"bf16_tflops_sustained {peak_src} (timed region {timed_s:.1f} s of "
                                     f"back-to-back launches)" if sustained else
                                     f"bf16_tflops {peak_src} (burst: timed region {timed_s:.2f} s)"),
                     "frac_of_burst": round(achieved / peak_burst, 4),
                     "kernel_ms": round(ms_kernel, 4), "flops_per_launch": flops_rank,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of the value variant's "
                                       "launch, ncu in this run" if traffic is not None else None},
        "by_mapping": by_mapping,
        "topology": {"n_domains": topo["n_domains"], "sms_per_domain": topo["sms_per_domain"],
                     "source": topo["source"], "lat_near_cyc": round(topo["lat_near_cyc"], 1),
                     "lat_far_cyc": round(topo["lat_far_cyc"], 1),
                     "far_lines_cached_near": topo["far_lines_cached_near"]},
        "e2e": {"value": round(flops_job / t_e2e / 1e12, 2), "unit": "TFLOP/s", "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": d2h * world, "ms_per_step": round(t_e2e * 1e3, 3),
                "api": e2e_api},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if ncu_prov is not None:
        out["ncu"] = ncu_prov
    if replicated is not None:
        out["replicated_output"] = replicated
    if rank == 0 and world == 1 and not a.no_cpu_baseline and a.pass_ == "fwd":
        out["cpu_baseline"] = cpu_baseline(a.workload, a.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def measure_replicated(api, pdist, qkvo, shard, full_shape, causal, scale, mapping, rank, world, dev, stream,
                       reps=5):
    import torch
    import torch.distributed as tdist

    q, k, v, o = qkvo
    dist_on = tdist.is_available() and tdist.is_initialized()

    def agree(ok):
        # every rank learns whether all ranks succeeded, so a failure on one
        # rank never leaves the others waiting in a collective below
        if not dist_on:
            return ok
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev if tdist.get_backend() == "nccl" else "cpu")
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
    nccl = dist_on and tdist.get_backend() == "nccl"

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
    gathered_out = [None]

    def gathered():
        api.attn_fwd(q, k, v, o, causal=causal, scale=scale, mapping=mapping, stream=stream)
        gathered_out[0] = pdist.all_gather_heads(o, world)

    def time_it(fn):
        ts = []
        for i in range(reps + 2):
            torch.cuda.synchronize()
            if dist_on:
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
           "fwd_then_allgather_ms": round(time_it(gathered), 4),
           "allgather_backend": tdist.get_backend() if dist_on else "none (one rank, no process group)",
           "o_bytes_per_rank": o.numel() * o.element_size(),
           "method": "attn_fwd_replicated: epilogue stores each O tile into all ranks' buffers (CUDA IPC, NVLink "
                     "P2P); vs attn_fwd + dist.all_gather_heads (all_gather_into_tensor under NCCL); median of "
                     f"{reps}, device events, max over ranks"}
    if nccl:
        res["fwd_then_nccl_allgather_ms"] = res["fwd_then_allgather_ms"]
    # the fused result must equal the gathered one (heads are independent)
    if dist_on:
        tdist.barrier()
    res["bit_identical"] = bool(torch.equal(po.local.view(torch.int16), gathered_out[0].view(torch.int16)))
    po.close()
    return res


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ----------------------------------------------------------- oracle (CPU)
def cpu_info():
    """Host CPU model, sockets and usable threads (lscpu; sched_getaffinity)."""
    info = {"threads": len(os.sched_getaffinity(0))}
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in txt.splitlines():
            k, _, v = line.partition(":")
            if k.strip() == "Model name":
                info["model"] = v.strip()
            elif k.strip() == "Socket(s)":
                info["sockets"] = int(v.strip()) if v.strip().isdigit() else v.strip()
    except Exception:  # noqa: BLE001
        pass
    return info


def sampled_heads(name, n_groups=2, seed=5):
    """Oracle inputs for a sample of whole KV groups of workload `name`: only
    those heads are generated (seeded per head exactly like the full tensors,
    synth.py), so a 16 GiB workload costs a few hundred MB on the host.
    Returns (shape of the sample, (q, k, v), description)."""
    import numpy as np

    from paper_2511_02132_b200 import synth

    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
    G = Hq // Hkv
    rng = np.random.default_rng(seed)
    pick = sorted({(int(rng.integers(0, B)), int(rng.integers(0, Hkv))) for _ in range(n_groups)})
    dtype = "fp32" if name == "C1" else "bf16"
    import torch

    tdt = torch.float32 if name == "C1" else torch.bfloat16
    qs, ks, vs = [], [], []
    for b, g in pick:
        q, k, v = synth.make_qkv(1, G, 1, N, d, base=0, q_head_offset=g * G, kv_head_offset=g, batch_offset=b,
                                 device="cpu", dtype=tdt)
        qs.append(q), ks.append(k), vs.append(v)
    q, k, v = (torch.cat(x, dim=1) for x in (qs, ks, vs))
    return (1, G * len(pick), len(pick), N, d, causal), (q, k, v), f"{len(pick)} KV group(s) {pick} ({dtype})"


def _rows(shape, n, seed):
    """Stratified query rows of a sample: i = 0, N-1, 128-row block edges,
    then uniform random (SURVEY.md §8(c) strata)."""
    import numpy as np

    B, Hq, _, N, _, _ = shape
    rng = np.random.default_rng(seed)
    edge = [0, N - 1] + [x for blk in rng.integers(0, max(1, N // 128), 8) for x in (blk * 128, blk * 128 + 127)]
    i = np.concatenate([np.clip(np.array(edge), 0, N - 1), rng.integers(0, N, max(0, n - len(edge)))])[:n]
    return np.stack([rng.integers(0, B, len(i)), rng.integers(0, Hq, len(i)), i], 1).astype(np.int64)


def _row_flops(shape, rows):
    _, _, _, N, d, causal = shape
    if causal:
        return float((4.0 * d * (rows[:, 2] + 1)).sum())
    return 4.0 * d * N * len(rows)


def _time_rows(oa, shape, qkv, seconds, threads, seed):
    """Time the oracle on as many stratified rows as fit in ~`seconds`."""
    q, k, v = qkv
    d, causal = shape[4], shape[5]
    scale = 1.0 / math.sqrt(d)
    oa.set_threads(threads)
    probe = _rows(shape, 8 * threads, 1)
    t0 = time.perf_counter()
    oa.attention_rows(q, k, v, probe, causal=causal, scale=scale)
    per_row = (time.perf_counter() - t0) / len(probe)
    n = int(max(threads, min(400000, seconds / max(per_row, 1e-9))))
    rows = _rows(shape, n, seed)
    t0 = time.perf_counter()
    oa.attention_rows(q, k, v, rows, causal=causal, scale=scale)
    dt = time.perf_counter() - t0
    fl = _row_flops(shape, rows)
    return fl / dt, n, dt, fl


def cpu_baseline(name, seconds):
    """The oracle as it stands, on this host's cores: a bounded stratified row
    sample of `name` (value, all threads), plus the per-core figures SURVEY
    §8(d) asks for -- single-thread C1 (full) and C2 (sampled rows) -- and the
    C1 fp32 full oracle ("CPU oracle in seconds", BASELINE.json config 1)."""
    from oracle import attn as oa

    info = cpu_info()
    threads = info["threads"]
    shape, qkv, desc = sampled_heads(name)
    rate, n, dt, fl = _time_rows(oa, shape, qkv, seconds, threads, 2)
    out = {"value": round(rate / 1e12, 6), "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
           "sample": f"{n} stratified query rows of {name} from {desc} (fp64 two-pass softmax, "
                     f"{fl / 1e9:.1f} GFLOP) in {dt:.1f} s, {threads} threads",
           "seconds": round(dt, 2), "cpu_model": info.get("model"), "sockets": info.get("sockets")}
    extra = {}
    try:  # C1 fp32, the whole problem, all threads and one thread
        from paper_2511_02132_b200 import synth

        B, Hq, Hkv, N, d, causal, _ = WORKLOADS["C1"]
        q1, k1, v1 = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cpu", dtype=__import__("torch").float32)
        for th in (threads, 1):
            oa.set_threads(th)
            t0 = time.perf_counter()
            oa.attention(q1, k1, v1, causal=causal, scale=1.0 / math.sqrt(d))
            extra[f"C1_fp32_full_{'1thread' if th == 1 else f'{th}threads'}_s"] = round(time.perf_counter() - t0, 6)
        # C2 sampled rows on one thread (per-core cost)
        s2, qkv2, desc2 = sampled_heads("C2", n_groups=1)
        r2, n2, dt2, _ = _time_rows(oa, s2, qkv2, min(4.0, seconds / 3), 1, 3)
        extra["C2_1thread_tflops"] = round(r2 / 1e12, 6)
        extra["C2_1thread_sample"] = f"{n2} rows of {desc2} in {dt2:.1f} s"
        extra["C2_full_extrapolated_1thread_s"] = round(flops_fwd(1, 32, 8192, 128, False) / r2, 1)
        extra["C2_full_extrapolated_all_threads_s"] = round(flops_fwd(1, 32, 8192, 128, False) / r2 / threads, 1)
    except Exception as e:  # noqa: BLE001
        extra["error"] = repr(e)[:200]
    oa.set_threads(threads)
    out["per_core"] = extra
    if name != "C1":
        B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
        out["full_extrapolated_s"] = round(flops_fwd(B, Hq, N, d, causal) / rate, 1)
        out["full_extrapolated_note"] = "sampled time / sampled flops x total flops (extrapolated)"
    return out


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle
    from oracle import attn as oa

    info = cpu_info()
    threads = info["threads"]
    shape, (q, k, v), desc = sampled_heads(a.workload)
    oa.set_threads(threads)
    scale = 1.0 / math.sqrt(shape[4])
    probe = _rows(shape, 4 * threads, 1)
    t0 = time.perf_counter()
    oa.attention_rows(q, k, v, probe, causal=shape[5], scale=scale)
    per_row = (time.perf_counter() - t0) / len(probe)
    budget = max(0.05, min(2.0, 90.0 / max(1, a.steps + a.warmup)))  # whole run within ~1.5 min
    n = int(max(threads, budget / max(per_row, 1e-9)))
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
    sample = f"{n} stratified query rows per step from {desc} of {a.workload} (fp64 two-pass softmax oracle)"
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(tot_t / a.steps * 1e3, 3),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (i.i.d. N(0,1) rounded to bf16, seeded per head)",
        "config": {"workload": a.workload, "B": B, "Hq": Hq, "Hkv": Hkv, "N": N, "d": d, "causal": causal,
                   "mapping": a.mapping, "parallelism": "CPU oracle on rank 0 host cores"},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu_model": info.get("model"), "sockets": info.get("sockets")},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--mapping", default="swizzled_head_first", choices=VARIANT_MAPS + ("swizzled_head_first:shared",))
    ap.add_argument("--order", default="ascending", choices=("ascending", "descending", "alternate"),
                    help="unit order of the value variant (ATTN_ORDER_*); by_mapping uses ascending")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-replicated", action="store_true",
                    help="skip the replicated-output (fused peer-store vs all-gather) measurement")
    ap.add_argument("--replicated", action="store_true",
                    help="measure replicated output even at one rank (process group of one, NCCL under torchrun)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sets", type=int, default=0, help="resident input sets rotated per step (0: auto)")
    ap.add_argument("--flush", action="store_true", help="memset a 2xL2 buffer before every step")
    ap.add_argument("--cluster", type=int, default=1, choices=(0, 1),
                    help="value variant as CTA-pair clusters with K/V multicast (ATTN_CLUSTER_MULTICAST, NEXT-4)")
    ap.add_argument("--ncu", default="auto", choices=("auto", "on", "off"),
                    help="per-variant ncu counters measured in this run by a child process (auto: forward)")
    ap.add_argument("--ncu-timeout", type=float, default=900.0)
    ap.add_argument("--pass", dest="pass_", default="fwd", choices=("fwd", "bwd"),
                    help="time the forward (default, the headline) or the backward (NEXT-3)")
    ap.add_argument("--ncu-child", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--variants", default="", help=argparse.SUPPRESS)
    ap.add_argument("--device", type=int, default=0, help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.ncu_child:
        ncu_child(a)
        return
    if a.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
