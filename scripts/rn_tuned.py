"""r_n family (NEXT-2): the default static HOT ranking against sfa_tune_residency on a
sample of the text.  usage: python scripts/rn_tuned.py [n ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1405_0562_b200 as P  # noqa: E402
import bench  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ns = [int(x) for x in sys.argv[1:]] or [20, 50, 100, 127]
    stream = torch.cuda.Stream()
    for n in ns:
        text = W.rn_accepted(n, 1 << 30)
        sfa = P.SFA(W.rn_regex(n), b"0123456789")
        dt = torch.from_numpy(text).cuda()
        res = torch.zeros(2, dtype=torch.int32, device="cuda")
        fn = lambda: sfa.match_async(dt, res, stream)  # noqa: E731
        ms0, _ = bench.steady(torch, fn, stream, 30, 3)
        r0 = res.cpu().tolist()
        sfa.tune_residency(dt[:8 << 20], stream)
        ms1, _ = bench.steady(torch, fn, stream, 30, 3)
        r1 = res.cpu().tolist()
        info = sfa.info()
        for knobs in os.environ.get("RN_TUNINGS", "").split(";"):
            if not knobs:
                continue
            sfa.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in knobs.split(","))})
            try:
                msk, _ = bench.steady(torch, fn, stream, 30, 3)
                i2 = sfa.info()
                print(f"   {knobs}: {text.size / msk / 1e6:.0f} GB/s {res.cpu().tolist()} copies {i2['dfa_window_copies']} hot {i2['dfa_window_hot']}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"   {knobs}: {e}", flush=True)
            sfa.set_tuning()
        print(f"r{n}: |D|={info['dfa_states']} |S|={info['sfa_states']} static {text.size / ms0 / 1e6:.0f} GB/s  "
              f"tuned {text.size / ms1 / 1e6:.0f} GB/s  results {r0} {r1} copies {info['dfa_window_copies']} hot {info['dfa_window_hot']}", flush=True)
        del dt
        sfa.close()


if __name__ == "__main__":
    main()
