"""Top SASS lines of one kernel by warp-stall samples, with their top stall
reasons, from `ncu -i REP --page source --csv --print-source sass` output.

    python scripts/ncu_sass_hot.py source.csv [N] [grep-pattern]
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
recs, tot = [], 0.0
for r in data:
    try:
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    tot += smp
    recs.append((smp, r))
print(f"{rows[0][1]}\ntotal warp-stall samples {tot:.0f}")
sel = [x for x in recs if pat is None or pat.search(x[1][ix["Source"]])]
for smp, r in sorted(sel, key=lambda x: -x[0])[:n]:
    st = sorted(((float(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{r[ix['Address']]:>16} {smp:8.0f} {100 * smp / tot:5.2f}%  {r[ix['Source']][:64]:64s} "
          + " ".join(f"{h}={v:.0f}" for v, h in st if v > 0))
