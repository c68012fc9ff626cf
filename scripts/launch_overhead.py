"""Host time per sfa_match_async call (ctypes + C-ABI + launch) and the
single-launch event time around it, cfg2 (256 MiB).  usage: python scripts/launch_overhead.py"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1405_0562_b200 as P  # noqa: E402

for cfg in (2, 3):
    rx, alpha, text = bench.workload(cfg)
    sfa = P.SFA(rx, alpha)
    dt = torch.from_numpy(text).cuda()
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    L = P.lib()
    for _ in range(5):
        sfa.match_async(dt, res, s)
    torch.cuda.synchronize()
    host, ev, raw = [], [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(30):
        torch.cuda.synchronize()
        e0.record(s)
        h0 = time.perf_counter()
        sfa.match_async(dt, res, s)
        h1 = time.perf_counter()
        e1.record(s)
        e1.synchronize()
        host.append(1e6 * (h1 - h0))
        ev.append(1e3 * e0.elapsed_time(e1))
    # the C call alone (no Python wrapper checks)
    args = (sfa.h, dt.data_ptr(), dt.numel(), s.cuda_stream, res.data_ptr())
    for _ in range(30):
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        L.sfa_match_async(*args)
        raw.append(1e6 * (time.perf_counter() - h0))
    torch.cuda.synchronize()
    print(f"cfg{cfg}: host per call {statistics.median(host):.1f} us (C call alone {statistics.median(raw):.1f} us), "
          f"event time {statistics.median(ev):.1f} us")
    sfa.close()
    del dt
