"""Static schedule of the forward kernel's unmasked softmax exp block from
cuobjdump SASS: sum of the control-code stall counts (the cycles one warp
needs to issue the block with no dynamic stalls) and the opcode histogram.
usage: python scripts/sass_static.py lib.so [D causal kCl]"""
import collections
import re
import subprocess
import sys

so = sys.argv[1]
D, causal, cl = (sys.argv[2:5] + ["128", "0", "1"][len(sys.argv[2:5]):]) if len(sys.argv) > 2 else ("128", "0", "1")
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
name = sys.argv[5] if len(sys.argv) > 5 else f"attn_fwd_sm100_kernelILi{D}ELb{causal}ELi{cl}E"
start = sass.index(name)
end = sass.find("Function :", start + 10)
lines = sass[start:end].split("\n")
ins = []
i = 0
while i < len(lines):
    m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", lines[i])
    if m:
        m2 = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        ins.append((int(m.group(1), 16), m.group(2).strip(), int(m2.group(1), 16)))
        i += 2
    else:
        i += 1
# blocks = maximal runs that contain MUFU.EX2 between STTM-bounded regions: take each
# STTM.x32 that stores P and walk back to the previous LDTM/branch target
mufu = [k for k, x in enumerate(ins) if "MUFU.EX2" in x[1]]
# cluster MUFU indices into blocks separated by > 200 instructions
blocks, cur = [], [mufu[0]]
for k in mufu[1:]:
    if k - cur[-1] > 120:
        blocks.append(cur)
        cur = [k]
    else:
        cur.append(k)
blocks.append(cur)
for b in blocks:
    if len(b) < 40:
        continue
    lo, hi = b[0] - 30, b[-1] + 30
    seg = ins[lo:hi]
    stall = sum((h >> 41) & 15 for _, _, h in seg)
    ops = collections.Counter()
    for _, t, _ in seg:
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        ops[op.split(".")[0]] += 1
    print(f"block @0x{seg[0][0]:x}: {len(b)} MUFU, {len(seg)} instrs, static stall sum {stall} cycles; "
          + ", ".join(f"{k} {v}" for k, v in ops.most_common(9)))
