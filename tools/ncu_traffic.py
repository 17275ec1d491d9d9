"""Per-config DRAM traffic of the FineGrainedCombined render kernel, read from
the committed ncu --set full summaries (profiles/r1_ncu_full_render_fine_exact*.txt),
written as profiles/ncu_traffic.json for bench.py's roofline "traffic" field.

  python tools/ncu_traffic.py profiles > profiles/ncu_traffic.json
"""
import json
import os
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(path):
    tot = 0.0
    for line in open(path):
        f = line.split()
        if f and f[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(f[1].replace(",", "")) * UNIT[f[2]]
    return int(round(tot))


d = sys.argv[1]
out = {}
for key, name in (("c2", "r1_ncu_full_render_fine_exact.txt"), ("c1", "r1_ncu_full_render_fine_exact_c1.txt"),
                  ("c4", "r1_ncu_full_render_fine_exact_c4.txt"),
                  ("c2_super", "r1_ncu_full_render_fine_super_c2.txt"),
                  ("c4_super", "r1_ncu_full_render_fine_super_c4.txt")):
    p = os.path.join(d, name)
    if os.path.exists(p):
        cfg, _, sup = key.partition("_")
        out[f"{cfg}_FineGrainedCombined_exact" + ("_super" if sup else "")] = dram_bytes(p)
        out[f"_source_{key}"] = (f"profiles/{name}: dram__bytes_read.sum + dram__bytes_write.sum, one {cfg} launch "
                                 "of bench's first view (ncu --set full, cold cache)")
print(json.dumps(out, indent=1))
