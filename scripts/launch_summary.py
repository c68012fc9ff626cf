"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
profiles/<tag>_launches.txt: every launch (kernel, ns) and totals by kernel.
usage: python scripts/launch_summary.py gpurun_out/<tag>_launches.csv profiles/<tag>_launches.txt "<command>" """
import collections
import csv
import re
import sys

src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
hdr, body = rows[0], rows[1:]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
launches = [(r[ik], float(r[iv].replace(",", ""))) for r in body if r[im] == "gpu__time_duration.sum"]
tot = collections.OrderedDict()
for k, v in launches:
    key = re.sub(r"\(.*$", "", k.replace("void ", "")) if not k.startswith("void sfa::k_scan_tma") else \
        k.replace("void ", "").split("(sfa::TmaMaps")[0]
    tot[key] = tot.get(key, 0.0) + v
all_ns = sum(v for _, v in launches)
with open(dst, "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, launch list of\n# %s\n" % cmd)
    f.write("# (cold-cache, serialised per launch: compare shares, not absolute times).  kernel, ns\n")
    for k, v in launches:
        f.write("%s, %d\n" % (k[:110], v))
    f.write("# totals by kernel (share of all device time in the list):\n")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write("#   %s: %.1f us (%.1f%%)\n" % (k[:120], v / 1e3, 100 * v / all_ns))
print(open(dst).read().split("# totals")[1])
