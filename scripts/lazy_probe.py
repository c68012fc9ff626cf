"""r_500 / r_a on the fly, factored chunk runs on and off: first match,
steady match (median of 5, host wall clock around the blocking call), states
and transitions built.  usage: python scripts/lazy_probe.py [MiB] [factored-only: 1]"""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1405_0562_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
modes = (0,) if len(sys.argv) > 2 and sys.argv[2] == "1" else (0, 1)
s = torch.cuda.Stream()
for name, rx, alpha, gen in (("r500", W.rn_regex(500), b"0123456789", lambda: W.rn_accepted(500, mib << 20)),
                             ("ra500", W.ra_regex(500), b"0123456789a", lambda: W.ra_text(mib << 20))):
    text = gen()
    dt = torch.from_numpy(text).cuda()
    for nf in modes:
        sfa = P.SFA(rx, alpha, lazy=True)
        sfa.set_tuning(no_factor=nf)
        t0 = time.perf_counter()
        r = sfa.match_lazy(dt, s)
        first = time.perf_counter() - t0
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            assert sfa.match_lazy(dt, s) == r
            ts.append(time.perf_counter() - t0)
        ms = 1e3 * statistics.median(ts)
        i = sfa.info()
        print(json.dumps({"regex": name, "no_factor": nf, "result": list(r), "first_s": round(first, 3),
                          "ms": round(ms, 3), "GBps": round(text.size / ms / 1e6, 1), "states": i["sfa_states"],
                          "transitions": i["lazy_transitions"], "host_build_s": round(i["lazy_seconds"], 3)}),
              flush=True)
        sfa.close()
