"""Diagnostic: force TMA shapes (SFA_TMA_CONFIG) on cfg2 texts of several sizes
and compare sfa_match / sfa_match_host with the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, paper_1405_0562_b200 as P, workloads as W

shapes = sys.argv[1].split(";") if len(sys.argv) > 1 else ["2,32,0"]
rx, al = W.REGEX[2], W.ALPHABET[2]
d = O.OracleDFA(rx, al)
a = W.cfg2_accepted(14_000_000)
for shape in shapes:
    os.environ["SFA_TMA_CONFIG"] = shape
    sfa = P.SFA(rx, al)
    for n in (64 << 20, (64 << 20) + 1000, 100_000_000, 130_000_000, 20_000_000, 5_000_000):
        t = a[:n]
        dt = torch.from_numpy(t).cuda()
        got = sfa.match(dt); exp = d.run(t)
        goth = sfa.match_host(t)
        print(shape, n, "match", got, "host", goth, "oracle", exp, "OK" if got == exp == goth else "MISMATCH", flush=True)
        if got != exp:
            # locate: chunked with SPEC rule is the direct kernel; bisect the prefix where the TMA path diverges
            lo, hi = 4 << 20, n
            while hi - lo > 4096:
                mid = (lo + hi) // 2
                if sfa.match(dt[:mid]) == d.run(t[:mid]): lo = mid
                else: hi = mid
            print("   first failing prefix length ~", hi, flush=True)
