"""Small invocations of every kernel for compute-sanitizer (memcheck, racecheck,
synccheck): the TMA scan (PRIVATE cfg2, HOT + FACTORED cfg3) on ~4.5 MiB texts,
the direct scan, a ragged and an equal-length batch (k_batch_plan + the
segmented scan), the sharded-map calls and Alg. 3.  Checks every result against
the oracle; exit 0 on success.  usage: python scripts/sanitize_case.py [small]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1405_0562_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = (4 << 20) + 4097
s = torch.cuda.Stream()
for rx, alpha, text in [("([0-4]{5}[5-9]{5})*", b"0123456789", W.cfg2_accepted(n // 10 + 1)[:n]),
                        (W.cfg3_regex(), None, W.cfg3_text(n, plant=True))]:
    d = O.OracleDFA(rx, alpha)
    sfa = P.SFA(rx, alpha)
    dt = torch.from_numpy(text).cuda()
    assert sfa.match(dt, s) == d.run(text), rx                         # k_scan_tma
    assert sfa.match(dt[:70_001], s) == d.run(text[:70_001])           # k_scan_direct
    texts, off = W.ragged_batch(3, 300, 30_000, alpha or b"abcdefghijklmnopqrstuvwxyz")
    res = torch.zeros(600, dtype=torch.int32, device="cuda")
    sfa.match_batch(torch.from_numpy(texts).cuda(), torch.from_numpy(off.astype(np.int64)).cuda(), 300, res, s)
    s.synchronize()
    got = res.cpu().numpy().view(np.uint32).reshape(300, 2)
    qo, ao = d.run_batch(texts, off)
    assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all()
    res = torch.zeros(2 * 64, dtype=torch.int32, device="cuda")
    sfa.match_batch_uniform(dt, 65536, 64, res, s)                      # equal texts
    s.synchronize()
    got = res.cpu().numpy().view(np.uint32).reshape(64, 2)
    qo, ao = d.run_batch(text[:64 * 65536], np.arange(65, dtype=np.uint64) * 65536)
    assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all()
    r1 = torch.zeros(2, dtype=torch.int32, device="cuda")
    sfa.match_speculative(dt[:300_000], r1, 0, None, s)                 # Alg. 3
    s.synchronize()
    assert tuple(r1.cpu().numpy().view(np.uint32)) == (d.run(text[:300_000])[0], int(d.run(text[:300_000])[1]))
    nd = sfa.info()["dfa_states"]
    maps = torch.zeros(2 * nd, dtype=torch.int32, device="cuda")
    h = text.size // 2
    sfa.match_map(dt[:h], maps[:nd], s)
    sfa.match_map(dt[h:], maps[nd:], s)
    sfa.combine_maps(maps, 2, r1, s)
    s.synchronize()
    assert tuple(r1.cpu().numpy().view(np.uint32)) == (d.run(text)[0], int(d.run(text)[1]))
    del dt
    sfa.close()
print("sanitize case ok")
