"""One config's hot call, `reps` times after 3 warm-ups (for ncu: -s 3 -c 1 or a launch list).
usage: python scripts/one_launch.py <cfg> [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1405_0562_b200 as P  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rx, alpha, text = bench.workload(cfg)
sfa = P.SFA(rx, alpha)
s = torch.cuda.Stream()
if cfg == 5:
    texts, off, _ = text
    dt = torch.from_numpy(texts).cuda()
    do = torch.from_numpy(off.astype(np.int64)).cuda()
    res = torch.zeros(2 * (off.size - 1), dtype=torch.int32, device="cuda")
    fn = lambda: sfa.match_batch(dt, do, off.size - 1, res, s)  # noqa: E731
else:
    dt = torch.from_numpy(text).cuda()
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    fn = lambda: sfa.match_async(dt, res, s)  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
for _ in range(reps):
    fn()
    torch.cuda.synchronize()
print("done", cfg, res[:2].cpu().tolist())
