"""Drive scripts/micro/l2_capacity.cu (see its header): effective L2 capacity
seen by ONE die vs BOTH dies of B200, and whether two dies reading the same
lines need the capacity twice (a near-die copy per die).  Event-timed here;
run under ncu (scripts/l2_capacity.sh) for DRAM bytes per launch.

    python scripts/l2_capacity.py [--mib 32,48,64,...] [--passes 8]
Analysis tooling only (not on the product path)."""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_topology  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "micro", "libl2cap.so")
ap = argparse.ArgumentParser()
ap.add_argument("--mib", default="16,32,48,56,64,72,80,96,112,128,160")
ap.add_argument("--passes", type=int, default=8)
ap.add_argument("--configs", default="die0_split,die1_split,both_split,both_each")
ap.add_argument("--json", default=None)
a = ap.parse_args()
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "micro", "l2_capacity.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", SO, os.path.join(HERE, "micro", "l2_capacity.cu")])
lib = ctypes.CDLL(SO)
lib.l2cap_run.restype = ctypes.c_float
lib.l2cap_run.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                          ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
t = attn_topology(0)
dom = torch.tensor(t["domain_of_smid"] + [-1] * (512 - len(t["domain_of_smid"])), dtype=torch.int8, device="cuda")
spd = (ctypes.c_int * 2)(*t["sms_per_domain"][:2])
buf = torch.ones(max(int(x) for x in a.mib.split(",")) << 20, dtype=torch.uint8, device="cuda")
flush = torch.empty(2 * t["l2_bytes"], dtype=torch.uint8, device="cuda")
CFG = {"die0_split": (1, 0), "die1_split": (2, 0), "both_split": (3, 0), "both_each": (3, 1)}
rows = []
print(json.dumps({k: t[k] for k in ("sms_per_domain", "l2_bytes", "lat_near_cyc", "lat_far_cyc",
                                     "lat_near_reread_cyc", "lat_far_reread_cyc", "far_lines_cached_near")}))
for mib in (int(x) for x in a.mib.split(",")):
    for name in a.configs.split(","):
        mask, mode = CFG[name]
        flush.zero_()
        torch.cuda.synchronize()
        ms = lib.l2cap_run(buf.data_ptr(), mib << 20, dom.data_ptr(), mask, mode, a.passes, t["num_sms"], spd)
        readers = 2 if mode == 1 else 1
        r = {"mib": mib, "config": name, "passes": a.passes, "ms": round(ms, 4),
             "l2_read_gbs": round(readers * a.passes * (mib << 20) / (ms * 1e-3) / 1e9, 1) if ms > 0 else None}
        rows.append(r)
        print(json.dumps(r), flush=True)
if a.json:
    json.dump(rows, open(a.json, "w"), indent=1)
