"""Run the die-topology probe and print/analyse it (dump raw latencies with ATTN_NUMA_PROBE_DUMP)."""
import json
import sys

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_topology

t = attn_topology(0)
d = t.pop("domain_of_smid")
print(json.dumps(t))
print("domain_of_smid:", "".join(str(x) if x >= 0 else "." for x in d))
