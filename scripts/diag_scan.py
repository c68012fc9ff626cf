"""Diagnostic (not a bench line): GB/s of sfa_match_async for one config at several
text sizes, to separate fixed per-launch costs from the per-byte rate.
    python scripts/diag_scan.py <cfg> <MiB,MiB,...> [steps]
Honours SFA_TMA_CONFIG / SFA_DIAG_STRIDE (results unchecked under the latter)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1405_0562_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

cfg = int(sys.argv[1])
sizes = [int(x) << 20 for x in sys.argv[2].split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
if cfg == 2:
    rx, al, gen = W.REGEX[2], W.ALPHABET[2], lambda n: W.cfg2_accepted(n // 10)
elif cfg == 4:
    rx, al, gen = W.REGEX[4], W.ALPHABET[4], W.cfg4_text
elif cfg == 1:
    rx, al, gen = W.REGEX[1], W.ALPHABET[1], W.cfg1_random
else:
    rx, al, gen = W.cfg3_regex(), None, lambda n: W.cfg3_text(n, plant=False)
sfa = P.SFA(rx, al)
big = gen(max(sizes))
dt = torch.from_numpy(big).cuda()
res = torch.zeros(2, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
for n in sizes:
    v = dt[:n]
    for _ in range(5):
        sfa.match_async(v, res, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        sfa.match_async(v, res, s)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"cfg{cfg} n={n >> 20} MiB: {ms * 1e3:.1f} us/step, {n / ms / 1e6:.1f} GB/s  "
          f"[{os.environ.get('SFA_TMA_CONFIG', 'auto')} diag={os.environ.get('SFA_DIAG_STRIDE', '-')}]", flush=True)
