"""Diagnostic: host-side cost per sfa_match_async call vs device time (cfg1, 1 MiB)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1405_0562_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

sfa = P.SFA(W.REGEX[1], W.ALPHABET[1])
for n in (1 << 20, 16 << 20):
    t = torch.from_numpy(W.cfg1_random(n)).cuda()
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(20):
        sfa.match_async(t, res, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 2000
    h0 = time.perf_counter()
    e0.record(s)
    for _ in range(k):
        sfa.match_async(t, res, s)
    e1.record(s)
    h1 = time.perf_counter()
    e1.synchronize()
    print(f"n={n >> 20} MiB: host {1e6 * (h1 - h0) / k:.2f} us/call, device {1e3 * e0.elapsed_time(e1) / k:.2f} us/call")
    # raw C call without the Python wrapper's argument checks
    L = P.lib()
    import ctypes as C
    ptr, rp, sp = t.data_ptr(), res.data_ptr(), s.cuda_stream
    h0 = time.perf_counter()
    for _ in range(k):
        L.sfa_match_async(sfa.h, ptr, n, sp, rp)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"   raw ctypes: host {1e6 * (h1 - h0) / k:.2f} us/call")
