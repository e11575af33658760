"""Summarise an ncu --set full report of the attention kernel into profiles/ JSON."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__cycles_elapsed.max",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "lts__t_sector_op_read_hit_rate.pct", "lts__t_sectors.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tmem.sum", "smsp__inst_executed_pipe_xu.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def summarize(rep, extra):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = dict(extra)
    out["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            v = vals[i].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            u = units[i]
            # normalise to bytes / seconds
            if isinstance(v, float) and u in ("Kbyte", "Mbyte", "Gbyte", "Tbyte"):
                v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
                u = "byte"
            if isinstance(v, float) and u in ("usecond", "us"):
                v *= 1e-6
                u = "s"
            if isinstance(v, float) and u in ("msecond", "ms"):
                v *= 1e-3
                u = "s"
            if isinstance(v, float) and u in ("nsecond", "ns"):
                v *= 1e-9
                u = "s"
            out[k] = v
            out[k + ".unit"] = u
    rb, wb = out.get("dram__bytes_read.sum"), out.get("dram__bytes_write.sum")
    out["dram_bytes_per_launch"] = (rb + wb) if isinstance(rb, float) and isinstance(wb, float) else None
    return out


if __name__ == "__main__":
    rep, dst = sys.argv[1], sys.argv[2]
    extra = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
    s = summarize(rep, extra)
    json.dump(s, open(dst, "w"), indent=1)
    print(dst, {k: s.get(k) for k in ("gpu__time_duration.sum", "lts__t_sector_hit_rate.pct", "dram_bytes_per_launch")})
