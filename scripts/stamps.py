"""Per-CTA phase times of the TMA scan from the diagnostic library
(libsfa_diag.so, -DSFA_STAMPS).  usage: python scripts/stamps.py [configs]"""
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the diagnostic library (built by `python -m paper_1405_0562_b200._build --diag`), set before the
# package reads SFA_LIB at import
os.environ["SFA_LIB"] = os.path.join(ROOT, "paper_1405_0562_b200", "_lib", "libsfa_diag.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1405_0562_b200 as P  # noqa: E402
import bench  # noqa: E402

L = P.lib()
L.sfa_diag_stamps.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
L.sfa_diag_counters.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]


def report(name, h, G):
    st = np.zeros(G * 16, np.uint64)
    assert L.sfa_diag_stamps(h, st.ctypes.data, st.size) == 0
    st = st.reshape(G, 16).astype(np.int64)
    live = st[:, 0] > 0
    st = st[live]
    smid = st[:, 6].copy()
    st[:, 6] = 0
    t0 = st[:, 0].min()
    rel = (st - t0) / 1e3
    rel[st == 0] = np.nan
    q = lambda c: (np.nanmin(rel[:, c]), np.nanmedian(rel[:, c]), np.nanmax(rel[:, c]))  # noqa: E731
    print(f"{name}: ctas={st.shape[0]}")
    for c, what in [(0, "entry"), (7, "first TMA issued"), (1, "tables built"), (2, "after pdl wait"), (15, "first stage done"),
                    (3, "rows scanned"), (8, "aux+tail done"), (9, "values"), (10, "warps folded"),
                    (4, "CTA folded"), (11, "last: ticket"), (12, "last: parts+tail"), (13, "last: final fold"), (14, "last: fold again"),
                    (5, "epilogue end")]:
        mn, md, mx = q(c)
        print(f"  {what:18s} min {mn:8.2f}  median {md:8.2f}  max {mx:8.2f} us")
    ctr = np.zeros(16, np.uint64)
    if hasattr(L, "sfa_diag_counters") and L.sfa_diag_counters(h, ctr.ctypes.data, 16) == 0:
        print("  counters: combine_fact %d  combine_ids %d  combine_slow %d  replay %d  mixed folds %d"
              % tuple(int(x) for x in ctr[:5]))
    scan = rel[:, 3] - rel[:, 2]
    print(f"  scan duration      min {np.nanmin(scan):.2f} median {np.nanmedian(scan):.2f} max {np.nanmax(scan):.2f}")
    order = np.argsort(scan)
    print("  slowest CTAs (cta, smid, us):", [(int(b), int(smid[b]), round(float(scan[b]), 1)) for b in order[-12:]])
    print("  fastest CTAs (cta, smid, us):", [(int(b), int(smid[b]), round(float(scan[b]), 1)) for b in order[:8]])
    by_sm = np.full(int(smid.max()) + 1, np.nan)
    by_sm[smid] = scan
    print("  scan us by smid:", " ".join(f"{x:.0f}" for x in by_sm))


def main():
    cfgs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "3", "4", "5"])]
    G = torch.cuda.get_device_properties(0).multi_processor_count
    s = torch.cuda.Stream()
    for cfg in cfgs:
        rx, alpha, text = bench.workload(cfg)
        sfa = P.SFA(rx, alpha)
        if os.environ.get("STAMPS_TUNING"):  # e.g. STAMPS_TUNING=fact_fold=1
            sfa.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in os.environ["STAMPS_TUNING"].split(","))})
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
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        fn()
        report(f"cfg{cfg} (isolated)", sfa.h, G)
        for _ in range(3):
            fn()
        report(f"cfg{cfg} (after back-to-back)", sfa.h, G)
        del dt
        sfa.close()


if __name__ == "__main__":
    main()
