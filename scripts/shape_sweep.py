"""Steady and single-launch GB/s of the TMA scan per launch shape (K, ROWB, ring).
usage: python scripts/shape_sweep.py [configs]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1405_0562_b200 as P  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "4", "3"])]
shapes = [dict(), dict(tma_k=1, tma_rowb=32), dict(tma_k=2, tma_rowb=16), dict(tma_k=1, tma_rowb=16),
          dict(tma_k=2, tma_rowb=32), dict(tma_k=1, tma_rowb=64), dict(tma_k=2, tma_rowb=16, tma_ring=4),
          dict(tma_k=2, tma_rowb=16, tma_ring=6)]
if os.environ.get("SWEEP") == "ring":
    shapes = [dict(), dict(tma_k=1, tma_rowb=32, tma_ring=2), dict(tma_k=1, tma_rowb=32, tma_ring=3),
              dict(tma_k=1, tma_rowb=32, tma_ring=5), dict(tma_k=1, tma_rowb=64, tma_ring=2),
              dict(tma_k=1, tma_rowb=16, tma_ring=4), dict(tma_k=1, tma_rowb=16, tma_ring=8)]
if os.environ.get("SWEEP") == "promo":
    shapes = [dict(), dict(tma_promo=64), dict(tma_promo=128), dict(tma_promo=256),
              dict(tma_k=1, tma_rowb=16, tma_promo=128), dict(tma_k=1, tma_rowb=16, tma_promo=256)]
if os.environ.get("SWEEP") == "factored":   # the FACTORED layouts (cfg3/5): u16 R=16 vs u8 R=32, K = 1 / 2
    shapes = [dict(), dict(hot_rows=400), dict(tma_k=2, tma_rowb=16, hot_rows=400),
              dict(tma_k=2, tma_rowb=16, hot_rows=200), dict(dfa_u8=1), dict(dfa_u8=1, hot_rows=400),
              dict(dfa_u8=1, tma_k=2, tma_rowb=16, hot_rows=400), dict(dfa_u8=1, tma_k=2, tma_rowb=16, hot_rows=100),
              dict(tma_k=1, tma_rowb=32, hot_rows=200), dict(dfa_u8=1, tma_k=1, tma_rowb=32, hot_rows=200)]
if os.environ.get("SWEEP") == "mixed":   # DFA window layouts of the FACTORED step (cfg3/5)
    shapes = [dict(), dict(dfa_layout=1), dict(dfa_layout=2, dfa_hot=64), dict(dfa_layout=2, dfa_hot=40),
              dict(dfa_layout=2, dfa_hot=16), dict(tma_k=1, tma_rowb=32), dict(tma_k=1, tma_rowb=32, hot_rows=200),
              dict(tma_k=2, tma_rowb=16, hot_rows=200), dict(dfa_u8=1)]
if os.environ.get("SWEEP") == "ring2":   # FACTORED: smem for the ring instead of SFA hot rows
    shapes = [dict(), dict(hot_rows=256), dict(hot_rows=64), dict(hot_rows=16), dict(tma_k=1, tma_rowb=16, hot_rows=64, tma_ring=4),
              dict(tma_k=1, tma_rowb=32, hot_rows=16), dict(tma_k=1, tma_rowb=32, hot_rows=64),
              dict(tma_k=1, tma_rowb=32, hot_rows=16, dfa_hot=56), dict(tma_k=1, tma_rowb=32, hot_rows=16, dfa_hot=48)]
if os.environ.get("SWEEP") == "base":    # the automatic shape against the two 1-row alternatives
    shapes = [dict(), dict(tma_k=1, tma_rowb=16), dict(tma_k=1, tma_rowb=32)]
if os.environ.get("SWEEP") == "k2":      # two rows per thread (ILP 2) with 32-byte stages, 2-deep ring
    shapes = [dict(), dict(tma_k=2, tma_rowb=32, hot_rows=16), dict(tma_k=2, tma_rowb=32, hot_rows=16, dfa_hot=40),
              dict(tma_k=2, tma_rowb=32, hot_rows=16, dfa_hot=24), dict(tma_k=1, tma_rowb=64, hot_rows=16),
              dict(tma_k=1, tma_rowb=64, hot_rows=16, dfa_hot=40)]
if os.environ.get("SWEEP") == "k2promo":  # two chains per thread on 16-byte stages, L2 promotion for whole lines
    shapes = [dict(), dict(tma_k=2, tma_rowb=16, tma_promo=128), dict(tma_k=2, tma_rowb=16, tma_promo=256),
              dict(tma_k=2, tma_rowb=16, tma_promo=128, hot_rows=16), dict(tma_k=2, tma_rowb=16, tma_promo=256, hot_rows=16)]
if os.environ.get("SWEEP") == "hot2":    # cfg2 through HOT + FACTORED (an 8 KB DFA window): room for two rows per thread
    H = P.RES_HOT_L2
    shapes = [dict(), dict(_res=H), dict(_res=H, tma_k=2, tma_rowb=32, tma_ring=3), dict(_res=H, tma_k=2, tma_rowb=32),
              dict(_res=H, tma_k=2, tma_rowb=16), dict(_res=H, tma_k=1, tma_rowb=32, tma_ring=6),
              dict(_res=H, tma_k=1, tma_rowb=64, tma_ring=3), dict(_res=H, tma_k=2, tma_rowb=64, tma_ring=2)]
s = torch.cuda.Stream()
for cfg in cfgs:
    rx, alpha, text = bench.workload(cfg)
    if cfg == 5:
        texts, off, _ = text
        dt = torch.from_numpy(texts).cuda()
        do = torch.from_numpy(off.astype(np.int64)).cuda()
        res = torch.zeros(2 * (off.size - 1), dtype=torch.int32, device="cuda")
        n = texts.size
    else:
        dt = torch.from_numpy(text).cuda()
        res = torch.zeros(2, dtype=torch.int32, device="cuda")
        n = text.size
    ref = None
    for sh in shapes:
        sfa = P.SFA(rx, alpha)
        try:
            sh = dict(sh)
            res_mode = sh.pop("_res", None)
            if sh:
                sfa.set_tuning(**sh)
            if res_mode is not None:
                sfa.set_residency(res_mode)
                sh["_res"] = res_mode
            fn = (lambda: sfa.match_batch(dt, do, off.size - 1, res, s)) if cfg == 5 else (lambda: sfa.match_async(dt, res, s))
            ms, med = bench.steady(torch, fn, s, 30, 5)
            one = bench.single(torch, fn, s, 10)
            got = res.cpu().numpy().tobytes()
            ok = ref is None or got == ref
            ref = ref or got
            print(json.dumps({"cfg": cfg, "shape": sh, "steady_gbs": round(n / ms / 1e6), "single_gbs": round(n / one / 1e6),
                              "residency": P.RES_NAMES[sfa.info()["residency"]], "same_result": ok,
                              "dfa_hot": sfa.info()["dfa_window_hot"], "dfa_copies": sfa.info()["dfa_window_copies"]}),
                  flush=True)
        except P.SFAError as e:
            print(json.dumps({"cfg": cfg, "shape": sh, "error": str(e)}), flush=True)
        sfa.close()
    del dt
