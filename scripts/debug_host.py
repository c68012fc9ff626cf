"""Diagnostic: sfa_match_host slicing with forced TMA shapes vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O, paper_1405_0562_b200 as P, workloads as W

rx, al = W.REGEX[2], W.ALPHABET[2]
d = O.OracleDFA(rx, al)
a = W.cfg2_accepted(21_000_000)
M = 64 << 20
for shape in sys.argv[1].split(";"):
    os.environ["SFA_TMA_CONFIG"] = shape
    sfa = P.SFA(rx, al)
    for n in (2 * M, 2 * M + 10, 2 * M + (3 << 20), 3 * M, M + (5 << 20), M + (3 << 20), 2 * M + (5 << 20)):
        t = a[:n]
        exp = d.run(t)
        res = [sfa.match_host(t) for _ in range(3)]
        print(shape, n, res, exp, "OK" if all(r == exp for r in res) else "MISMATCH", flush=True)
