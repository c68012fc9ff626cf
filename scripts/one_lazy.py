"""The on-the-fly r_500 (or r_a) match, repeated (for ncu: -k regex:k_lazy_scan -s 4 -c 1).
usage: python scripts/one_lazy.py [r500|ra500] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_0562_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "r500"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if name == "r500":
    rx, alpha, text = W.rn_regex(500), b"0123456789", W.rn_accepted(500, 1 << 30)
else:
    rx, alpha, text = W.ra_regex(500), b"0123456789a", W.ra_text(1 << 30)
dt = torch.from_numpy(text).cuda()
sfa = P.SFA(rx, alpha, lazy=True)
s = torch.cuda.Stream()
print("first", sfa.match_lazy(dt, s), flush=True)
for _ in range(reps):
    t0 = time.perf_counter()
    r = sfa.match_lazy(dt, s)
    print("match", r, "%.3f ms" % (1e3 * (time.perf_counter() - t0)), flush=True)
