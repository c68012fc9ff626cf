"""bench.py -- GB/s of text matched on B200 (SFA run + composition), % of roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A step is one pass of the whole hot path (Alg. 5 of PAPER.md:552-576: byte ->
column, chunk runs from f_I, composition f_1 . ... . f_p, finalisation) over
one batch of the workload through the C-ABI, inputs resident in HBM.

Default workload (the headline): BASELINE.json configs[4] = cfg5, the largest
single-GPU configuration -- cfg3's 32-word contains-match DFA over 65,536
texts of 64 KiB (4 GiB) -- through north_star's ``sfa_match_batch`` (device
offsets; one k_batch_plan + one segmented k_scan_tma launch per step).  The
texts (4 GiB) are far larger than the 126 MB L2, so no flush is needed.

Beside it, on rank 0:
  * ``uniform_api``: the same batch through ``sfa_match_batch_uniform`` (host
    plan: the scan kernel alone);
  * ``per_config``: cfg2 (256 MiB), cfg3 and cfg4 (1 GiB) through
    ``sfa_match_async``, each with its roofline, the back-to-back step time
    (mean and median of the per-step events) and the single-launch time
    (launch to result, synchronised before each launch, median of >= 10);
  * ``single_launch`` of the headline itself;
  * ``cpu_baseline``: the oracle (Alg. 2, oracle/) on a bounded sample of the
    same workload on one host core, with nproc and the CPU model;
  * ``e2e``: the same batch end to end from pinned host memory through
    ``sfa_match_batch_host`` (H2D of texts and offsets, D2H of the results in
    the timed region);
  * ``per_config.ex3_n11``: the paper's Ex. 3 matched with the N-SFA (built
    from the NFA) beside the D-SFA;
  * ``per_config.on_the_fly_r500_ra``: r_500 and r_a (1 GiB) with the D-SFA
    built on the fly while matching, Alg. 3 beside.
``--spec`` adds the paper's baseline (Alg. 3) on cfg2-4; ``--rn`` the r_n
family; ``--shard`` one text over the ranks.

Multi-GPU (torchrun): every rank matches its own copy of the workload
(independent problems, no data-path collective), weak scaling; value = all
ranks' bytes / the max over ranks of the device time.

``--impl reference``: there is no reference implementation (the paper ships no
code); the reference arm is the CPU oracle (Alg. 2, oracle/) timed on the host
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GB/s of text matched on 1 B200 (SFA run + composition); % of roofline"
UNIT = "GB/s"
HBM_SPEC_GBS = 8000.0
CONFIG_NAMES = {
    1: "cfg1: (ab|ba)*c over {a,b,c}, 1 MiB accepted text",
    2: "cfg2: ([0-4]{5}[5-9]{5})* over digits, 268,435,450-byte accepted text",
    3: "cfg3: .*(w1|...|w32).* over all bytes, 1 GiB scrubbed a-z text, one planted word",
    4: "cfg4: .*a[ab]{8} over {a,b}, 1 GiB i.i.d. text",
    5: "cfg5: cfg3's DFA, batch of 65,536 x 64 KiB texts (4 GiB), 10% planted, through sfa_match_batch",
}
EXPECTED = {1: (3, True), 2: (0, True)}


def workload(cfg: int):
    """(regex, alphabet, text or (texts, offsets, planted)) of a BASELINE.json config."""
    import workloads as W
    if cfg == 1:
        return W.REGEX[1], W.ALPHABET[1], W.cfg1_accepted()
    if cfg == 2:
        return W.REGEX[2], W.ALPHABET[2], W.cfg2_accepted()
    if cfg == 3:
        return W.cfg3_regex(), None, W.cfg3_text(plant=True)
    if cfg == 4:
        return W.REGEX[4], W.ALPHABET[4], W.cfg4_text()
    if cfg == 5:
        return W.cfg3_regex(), None, W.cfg5_batch()
    raise ValueError(cfg)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)", {}


def host_info():
    model = "?"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count(), model


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (an nvidia-smi loop is too coarse for a ~0.1 s region)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.mx = [], set(), None
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.hdl = N.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(self.hdl, N.NVML_CLOCK_SM))
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.sm.append(float(N.nvmlDeviceGetClockInfo(self.hdl, N.NVML_CLOCK_SM)))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.hdl)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "NVML, 2 ms period, during the timed region"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def ncu_entry(key: str) -> dict:
    """The committed ncu --set full summary of the dominant kernel (profiles/ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f).get(key, {})
    except Exception:
        return {}


def ncu_traffic(key: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    return ncu_entry(key).get("dram_bytes_per_launch")


# --------------------------------------------------------------------------- timing
def steady(torch, fn, stream, steps, warmup):
    """K back-to-back steps on `stream`: (mean ms over the bracketing events, median of per-step events)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        fn()
        ev[i + 1].record(stream)
    ev[-1].synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return ev[0].elapsed_time(ev[-1]) / steps, statistics.median(per)


def single(torch, fn, stream, reps):
    """Launch-to-result device time of one isolated call (the device idle before
    it: no overlap with a previous launch), median of `reps`."""
    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def smem_peaks(nsm, sm_mhz):
    """Shared-memory ceilings: one conflict-free LDS wavefront per
    32 lookups -> 32 B/clk/SM; with the staged text (TMA write + LDS.128 read,
    1/128 wavefront each per byte) -> 21.33 B/clk/SM."""
    hz = sm_mhz * 1e6
    return nsm * 32 * hz / 1e9, nsm * (1.0 / (1 / 32 + 2 / 128)) * hz / 1e9


def pattern_ceiling():
    """GB/s of the scan's TMA access pattern (32-byte row pieces) without lookups: the best ring
    depth of the committed microbenchmark output."""
    try:
        best = 0.0
        with open(os.path.join(ROOT, "profiles", "r2d_mb_tma_ring.txt")) as f:
            for line in f:
                if "ROWB=32" in line and "GB/s" in line:
                    best = max(best, float(line.split(":")[1].split("GB/s")[0]))
        return best or None
    except Exception:
        return None


def roofline(gbs, peak, peak_kind, nsm, sm_mhz, kernel, traffic, per_launch_bytes, key=None):
    lk, dp = smem_peaks(nsm, sm_mhz)
    extra = {}
    e = ncu_entry(key) if key else {}
    if e.get("smem_wavefronts_ld"):
        # the shared-memory load data path at the measured wavefronts per byte (bank conflicts
        # included): one wavefront per SM per clock -> bytes * nsm * f / wavefronts
        ceil = per_launch_bytes * nsm * sm_mhz * 1e6 / e["smem_wavefronts_ld"] / 1e9
        extra = {"smem_ld_ceiling_gbs": ceil, "frac_of_smem_ld_ceiling": gbs / ceil,
                 "smem_conflicts_per_wavefront": e.get("smem_bank_conflicts_ld", 0) / e["smem_wavefronts_ld"],
                 "smem_ld_ceiling_source": "profiles/ncu_summary.json wavefronts of the same kernel"}
    pat = pattern_ceiling()
    if pat:
        extra.update({"access_pattern_ceiling_gbs": pat, "frac_of_access_pattern_ceiling": gbs / pat,
                      "access_pattern_ceiling_source": "profiles/r2d_mb_tma_ring.txt, best ring depth (scripts/mb_tma.cu: "
                                                       "k_scan_tma's TMA pattern on 1 GiB with the lookups removed; "
                                                       "context, measured in another session)"})
    return {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, **extra,
            "traffic": traffic, "traffic_source": "profiles/ncu_summary.json (ncu --set full of the same kernel)",
            "algorithmic_bytes_per_launch": per_launch_bytes,
            "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
            "frac_of_spec_8tbs": gbs / HBM_SPEC_GBS, "kernel": kernel,
            "smem_lookup_peak_gbs": lk, "smem_datapath_peak_gbs": dp, "sm_mhz_for_smem_peaks": sm_mhz,
            "frac_of_min_roofline": gbs / min(peak, lk), "frac_of_min_datapath": gbs / min(peak, dp)}


# --------------------------------------------------------------------------- CPU oracle
def cpu_sample(cfg, rx, alpha, text, budget_s):
    """The oracle (Alg. 2) on a bounded sample of the workload, one host core."""
    import oracle as O
    d = O.OracleDFA(rx, alpha)
    if cfg == 5:
        texts, off, _ = text
        k = 1024                                            # 64 MiB: the first 1,024 texts
        sample, soff = texts[: int(off[k])], off[: k + 1].copy()
        run = lambda: d.run_batch(sample, soff)           # noqa: E731
        what = f"the first {k} texts ({sample.size} bytes) of the cfg5 batch"
    else:
        sample = text[: min(text.size, 64 << 20)]
        run = lambda: d.run(sample)                        # noqa: E731
        what = f"the first {sample.size} bytes of the cfg{cfg} text"
    run()
    done, passes, t0 = 0, 0, time.perf_counter()
    while True:
        run()
        done += sample.size
        passes += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    el = time.perf_counter() - t0
    nproc, model = host_info()
    return {"value": done / el / 1e9, "unit": UNIT, "cores": 1, "nproc": nproc, "cpu_model": model, "kind": "oracle",
            "sample": f"{passes} passes over {what} ({el:.1f} s), Alg. 2 byte-at-a-time, single thread"}


def run_reference(args, world, rank):
    """CPU oracle (Alg. 2) on the host cores: the reference arm of this tier."""
    if rank != 0:
        return
    import oracle as O
    cfg = args.config
    rx, alpha, text = workload(cfg)
    d = O.OracleDFA(rx, alpha)
    if cfg == 5:
        texts, off, _ = text
        k = max(1, min(off.size - 1, args.ref_bytes // int(off[1] - off[0])))
        sample, soff = texts[: int(off[k])], off[: k + 1].copy()
        run = lambda: d.run_batch(sample, soff)   # noqa: E731
        what = f"the first {k} texts ({sample.size} bytes) of the cfg5 batch per step"
        nbytes = sample.size
    else:
        sample = text[: min(text.size, args.ref_bytes)]
        run = lambda: d.run(sample)               # noqa: E731
        what = f"the first {sample.size} bytes of the cfg{cfg} text per step"
        nbytes = sample.size
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    gbs = nbytes * len(times) / tot / 1e9
    nproc, model = host_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded, DESIGN.md input recipe)",
        "config": {"workload": CONFIG_NAMES[cfg], "bytes_per_step": int(nbytes)},
        "cpu_baseline": {"value": gbs, "unit": UNIT, "cores": 1, "nproc": nproc, "cpu_model": model, "kind": "oracle",
                         "sample": f"{what}, Alg. 2 byte-at-a-time (oracle/oracle.c)"},
        "e2e": {"value": gbs, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- per-config (single texts)
def spec_compare(torch, sfa, dtext, nbytes, sfa_ms, stream, warmup, expected):
    """Alg. 3 beside the SFA on one text: GB/s, lookups per byte, and the SFA's speedup."""
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    nd = sfa.info()["dfa_states"]
    steps = max(1, min(50, int(0.5 / max(1e-6, nbytes * nd / 5e12))))
    fn = lambda: sfa.match_speculative(dtext, res, 0, None, stream)  # noqa: E731
    ms, med = steady(torch, fn, stream, steps, min(warmup, 3))
    got = tuple(int(x) for x in res.cpu().numpy().view(np.uint32))
    if expected is not None and got != (expected[0], int(expected[1])):
        raise SystemExit(f"speculative result {got} != {expected}")
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"value": gbs, "unit": UNIT, "ms_per_step": ms, "steps": steps, "lookups_per_byte": nd,
            "lookups_per_s": gbs * 1e9 * nd, "sfa_speedup": ms / sfa_ms,
            "kernel": "k_spec_scan (Alg. 3, PAPER.md:293-328: the DFA from every state per chunk)"}


def single_text_config(torch, P, cfg, stream, steps, warmup, reps, peak, peak_kind, nsm, sm_mhz, spec=False,
                       text_in=None, nsfa=False):
    rx, alpha, text = workload(cfg) if text_in is None else text_in
    sfa = P.SFA(rx, alpha, nsfa=nsfa)
    dt = torch.from_numpy(text).cuda()
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    q, acc = sfa.match(dt, stream)
    if cfg in EXPECTED and (q, acc) != EXPECTED[cfg]:
        raise SystemExit(f"cfg{cfg}: wrong result {(q, acc)}")
    fn = lambda: sfa.match_async(dt, res, stream)  # noqa: E731
    ms, med = steady(torch, fn, stream, steps, warmup)
    one = single(torch, fn, stream, reps)
    n = text.size
    gbs = n / (ms * 1e-3) / 1e9
    info = sfa.info()
    out = {"workload": CONFIG_NAMES.get(cfg, rx), "bytes": int(n), "result": [q, bool(acc)],
           "value": gbs, "unit": UNIT, "ms_per_step": ms, "median_ms_per_step": med, "steps": steps,
           "single_launch": {"ms": one, "gbs": n / (one * 1e-3) / 1e9, "frac": n / (one * 1e-3) / 1e9 / peak,
                             "reps": reps, "how": "synchronised before each launch; launch-to-result events; median"},
           "roofline": roofline(gbs, peak, peak_kind, nsm, sm_mhz, "k_scan_tma (one launch per step)",
                                ncu_traffic(f"cfg{cfg}") if cfg else None, int(n), f"cfg{cfg}" if cfg else None),
           "residency": P.RES_NAMES.get(info["residency"], "?"), "sfa_states": info["sfa_states"],
           "dfa_states": info["dfa_states"], "api": "sfa_match_async", "gpu_launches_per_step": 1}
    if spec:
        out["alg3_speculative"] = spec_compare(torch, sfa, dt, n, ms, stream, warmup, (q, acc))
    del dt
    sfa.close()
    return out


def nsfa_compare(torch, P, stream, steps, warmup, reps, peak, peak_kind, nsm, sm_mhz, n=11, nbytes=1 << 30):
    """the paper's Ex. 3, matched with the
    N-SFA built from the NFA (sfa_compile_nsfa) beside the D-SFA of its minimal
    DFA (2^n states); both through the same kernels (1 GiB i.i.d. {a,l,p})."""
    import workloads as W
    rx, text = W.ex3_regex(n), W.ex3_text(n, nbytes)
    out = {}
    for name, nsfa in (("nsfa", True), ("dsfa", False)):
        sfa = P.SFA(rx, b"alp", nsfa=nsfa)
        info = sfa.info()
        r = single_text_config(torch, P, 0, stream, steps, warmup, reps, peak, peak_kind, nsm, sm_mhz,
                               text_in=(rx, b"alp", text), nsfa=nsfa)
        r.update({"workload": f"Ex. 3, n = {n}: {rx} over {{a,l,p}}, 1 GiB i.i.d. text", "kind": name,
                  "nfa_states": info["nfa_states"], "construction_s": info["dfa_seconds"] + info["sfa_seconds"]})
        out[name] = r
        sfa.close()
    return out


def lazy_family(torch, P, stream, warmup, peak, nbytes):
    """the paper's r_500 (|S| = 1,000,999) and r_a
     with the D-SFA built on the fly while matching
    (PAPER.md:532-542): the first match (construction + scan), the steady match
    of the same text (sfa_match_lazy, blocking), the states built, and Alg. 3
    (the speculative DFA, 1001 lookups per byte) on the same text beside it.
    Default: factored chunk runs (C24); "full_construction" repeats
    it with tuning no_factor, i.e. every visited state built (Table III's
    construction)."""
    import workloads as W
    out = {}

    def one(sfa, dt, size):
        t0 = time.perf_counter()
        q, acc = sfa.match_lazy(dt, stream)
        first_s = time.perf_counter() - t0
        times = []
        for _ in range(5):
            t0 = time.perf_counter()
            assert sfa.match_lazy(dt, stream) == (q, acc)
            times.append(time.perf_counter() - t0)
        ms = 1e3 * statistics.median(times)
        info = sfa.info()
        return (q, acc), {"states_built": info["sfa_states"], "transitions_built": info["lazy_transitions"],
                          "first_match_s": first_s, "host_build_s": info["lazy_seconds"],
                          "value": size / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms}

    for name, rx, alpha, gen in (("r500", W.rn_regex(500), b"0123456789", lambda: W.rn_accepted(500, nbytes)),
                                 ("ra500", W.ra_regex(500), b"0123456789a", lambda: W.ra_text(nbytes))):
        text = gen()
        dt = torch.from_numpy(text).cuda()
        sfa = P.SFA(rx, alpha, lazy=True)
        res, r = one(sfa, dt, text.size)
        if not res[1]:
            raise SystemExit(f"{name}: the accepted text was rejected ({res})")
        full = P.SFA(rx, alpha, lazy=True)
        full.set_tuning(no_factor=1)
        res_f, rf = one(full, dt, text.size)
        assert res_f == res
        full.close()
        info = sfa.info()
        r.update({"regex": f"{rx[:24]}...", "bytes": int(text.size), "dfa_states": info["dfa_states"],
                  "full_sfa_states": 1_000_999 if name == "r500" else 1_001_000,
                  "roofline_frac": r["value"] / peak, "mode": "factored chunk runs (C24)",
                  "timer": "host wall clock around the blocking call (median of 5)",
                  "full_construction": rf,
                  "alg3_speculative": spec_compare(torch, sfa, dt, text.size, r["ms_per_step"], stream, warmup, res)})
        out[name] = r
        del dt
        sfa.close()
    return out


def rn_family(torch, P, stream, warmup, peak, nbytes):
    """SURVEY 8(f) NEXT-2, the paper's scalability study on the GPU:
    r_n on an accepted text and r_a on "a"^m, the SFA beside Alg. 3 (speculative DFA)."""
    import workloads as W
    out = {}
    cases = [(f"r{n}", W.rn_regex(n), b"0123456789", lambda n=n: W.rn_accepted(n, nbytes))
             for n in (5, 10, 20, 50, 100, 127)]
    cases.append(("ra127", W.ra_regex(127), b"0123456789a", lambda: W.ra_text(nbytes)))
    for name, rx, alpha, gen in cases:
        text = gen()
        sfa = P.SFA(rx, alpha)
        dt = torch.from_numpy(text).cuda()
        res = torch.zeros(2, dtype=torch.int32, device="cuda")
        q, acc = sfa.match(dt, stream)
        if not acc:
            raise SystemExit(f"{name}: the accepted text was rejected ({q})")
        fn = lambda: sfa.match_async(dt, res, stream)  # noqa: E731
        ms, _ = steady(torch, fn, stream, 50, warmup)
        gbs = text.size / (ms * 1e-3) / 1e9
        info = sfa.info()
        out[name] = {"regex": rx, "bytes": int(text.size), "dfa_states": info["dfa_states"],
                     "sfa_states": info["sfa_states"], "residency": P.RES_NAMES.get(info["residency"], "?"),
                     "value": gbs, "unit": UNIT, "ms_per_step": ms, "roofline_frac": gbs / peak,
                     "alg3_speculative": spec_compare(torch, sfa, dt, text.size, ms, stream, warmup, (q, acc))}
        del dt
        sfa.close()
    return out


# --------------------------------------------------------------------------- headline: a batch
def bench_batch(args, torch, P, stream, world, rank, local, peak, peak_kind, nsm):
    rx, alpha, (texts, off, planted) = workload(5)
    count = off.size - 1
    sfa = P.SFA(rx, alpha)
    with torch.cuda.stream(stream):
        dt = torch.from_numpy(texts).cuda()
        do = torch.from_numpy(off.astype(np.int64)).cuda()
        res = torch.zeros(2 * count, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    fn = lambda: sfa.match_batch(dt, do, count, res, stream)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    r = res.view(count, 2).cpu().numpy().view(np.uint32)
    acc_idx = np.flatnonzero(r[:, 1])
    if acc_idx.tolist() != planted.tolist():              # exact: the planted texts and no other
        raise SystemExit("cfg5: the accepted texts are not exactly the planted ones")
    ref = res.clone()
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            fn()
            ev[i + 1].record(stream)
        ev[-1].synchronize()
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    ms = ev[0].elapsed_time(ev[-1])
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    if not torch.equal(ref, res):
        raise SystemExit("cfg5: results changed between steps")
    ms_per_step = ms / args.steps
    n = texts.size
    per_rank_gbs = n / (ms_per_step * 1e-3) / 1e9
    extra = {}
    if rank == 0:
        one = single(torch, fn, stream, args.single_reps)
        extra["single_launch"] = {"ms": one, "gbs": n / (one * 1e-3) / 1e9, "frac": n / (one * 1e-3) / 1e9 / peak,
                                  "reps": args.single_reps,
                                  "how": "synchronised before each call (k_batch_plan + k_scan_tma); median"}
        ufn = lambda: sfa.match_batch_uniform(dt, int(off[1] - off[0]), count, res, stream)  # noqa: E731
        ums, umed = steady(torch, ufn, stream, max(5, args.steps // 2), 3)
        if not torch.equal(ref, res):
            raise SystemExit("cfg5: sfa_match_batch_uniform differs from sfa_match_batch")
        extra["uniform_api"] = {"api": "sfa_match_batch_uniform (host plan; the scan kernel alone)",
                                "value": n / (ums * 1e-3) / 1e9, "ms_per_step": ums, "median_ms_per_step": umed}
    # end to end from pinned host memory through the library's host call: every
    # rank runs it at the same time on its own replica (barrier before, max over
    # ranks of the per-rank wall time), so the N-GPU value is measured, not scaled
    if args.e2e_steps > 0:
        htexts = torch.from_numpy(texts).pin_memory()
        hoff = torch.from_numpy(off.view(np.int64)).pin_memory()
        hres = torch.zeros(2 * count, dtype=torch.int32).pin_memory()
        sfa.match_batch_host(htexts, hoff, count, hres, stream)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            sfa.match_batch_host(htexts, hoff, count, hres, stream)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        if not torch.equal(hres, ref.cpu()):
            raise SystemExit("cfg5: sfa_match_batch_host differs")
        del htexts
        extra["e2e"] = {"value": world * n / e2e_s / 1e9, "unit": UNIT,
                        "h2d_bytes_per_step": int(n + off.nbytes), "d2h_bytes_per_step": int(8 * count),
                        "api": "sfa_match_batch_host (pinned host texts/offsets; slices of whole texts copied "
                               "on a copy stream while the previous slice is matched; results read back)",
                        "timer": "host wall clock around the blocking call"
                                 + (" (all ranks at once, max over ranks)" if world > 1 else ""),
                        "steps": args.e2e_steps}
    info = sfa.info()
    med = statistics.median(per)
    return sfa, dt, {
        "value": world * per_rank_gbs, "ms_per_step": ms_per_step, "per_rank_gbs": per_rank_gbs,
        "median_ms_per_step": med, "clocks": clk.summary(), "bytes": n, "count": count,
        "accepted": int(acc_idx.size), "residency": P.RES_NAMES.get(info["residency"], "?"),
        "sfa_states": info["sfa_states"], "dfa_states": info["dfa_states"], "wl": (rx, alpha, (texts, off, planted)),
        **extra}


def bench_sharded(args, torch, P, stream, world, rank, local, peak, peak_kind):
    """--shard: ONE text split over the ranks (strong scaling).  Per step every
    rank runs sfa_match_map on its shard, the ranks all-gather the |D|-entry
    mappings (NCCL) and fold them in text order (sfa_combine_maps)."""
    from paper_1405_0562_b200 import parallel as PL
    cfg = args.config if args.config != 5 else 2
    rx, alpha, text = workload(cfg)
    sfa = P.SFA(rx, alpha)
    a, b = PL.shard_bounds(text.size, world, rank)
    nD = sfa.info()["dfa_states"]
    with torch.cuda.stream(stream):
        dshard = torch.from_numpy(text[a:b]).cuda()
        local_map = torch.empty(nD, dtype=torch.int32, device="cuda")
        res = torch.zeros(2, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()

    def step():
        with torch.cuda.stream(stream):
            sfa.match_map(dshard, local_map, stream)
            maps = PL.gather_maps(local_map) if world > 1 else local_map.view(1, -1)
            sfa.combine_maps(maps, maps.shape[0], res, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    q, acc = res.cpu().tolist()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    gbs = text.size / (ms_per_step * 1e-3) / 1e9
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": gbs, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic (seeded, DESIGN.md input recipe)",
        "config": {"workload": CONFIG_NAMES[cfg], "bytes_per_step": int(text.size),
                   "parallelism": f"text sharded over {world} ranks; |D|-entry map all-gather (NCCL)",
                   "result": [q, bool(acc)]},
        "roofline": {"bound": "hbm", "achieved": gbs / world, "peak": peak, "unit": "GB/s",
                     "frac": gbs / world / peak, "traffic": None, "peak_kind": f"{peak_kind} copy bandwidth (per GPU)"},
        "clocks": clk.summary(), "gpu_launches": 2 * args.steps,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5, help="5 (default): the batch headline; 1-4: one text")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--per-config", default="2,3,4", help="single-text configs timed beside the headline ('' = none)")
    ap.add_argument("--single-reps", type=int, default=15)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-bytes", type=int, default=64 << 20)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", action="store_true", help="split ONE text over the ranks (strong scaling)")
    ap.add_argument("--rn", action="store_true",
                    help="also run the r_n scalability family (r5..r127, r_a) with Alg. 3 beside it")
    ap.add_argument("--rn-bytes", type=int, default=1 << 30)
    ap.add_argument("--no-lazy", dest="lazy", action="store_false",
                    help="skip r_500 and r_a with the D-SFA built on the fly (Alg. 3 beside)")
    ap.add_argument("--no-nsfa", dest="nsfa", action="store_false",
                    help="skip the N-SFA vs D-SFA line on the paper's Ex. 3")
    ap.add_argument("--spec", action="store_true",
                    help="also time the paper's baseline, Alg. 3 (speculative DFA), on each per-config text")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()

    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import paper_1405_0562_b200 as P
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak, peak_kind, peaks = load_peaks()
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    stream = torch.cuda.Stream()
    if args.shard:
        return bench_sharded(args, torch, P, stream, world, rank, local, peak, peak_kind)

    cfg = args.config
    if cfg == 5:
        sfa, dkeep, h = bench_batch(args, torch, P, stream, world, rank, local, peak, peak_kind, nsm)
        nbytes, api, launches = h["bytes"], "sfa_match_batch (device offsets; k_batch_plan + segmented k_scan_tma)", 2
        kernel = "k_batch_plan + k_scan_tma<SEG> (achieved = text bytes / step time, both launches included)"
        cfgd = {"workload": CONFIG_NAMES[5], "bytes_per_step": int(nbytes), "texts": h["count"],
                "accepted": h["accepted"], "l2": "4 GiB input > 126 MB L2: no flush needed", "api": api,
                "residency": h["residency"], "sfa_states": h["sfa_states"], "dfa_states": h["dfa_states"],
                "parallelism": f"replicas x{world}"}
        rx, alpha, wl = h.pop("wl")
        del dkeep
        sfa.close()
    else:
        rx, alpha, text = workload(cfg)
        per_rank = single_text_config(torch, P, cfg, stream, args.steps, args.warmup, args.single_reps, peak,
                                      peak_kind, nsm, peaks.get("sm_max_mhz", 1965.0), text_in=(rx, alpha, text))
        h = {"value": world * per_rank["value"], "ms_per_step": per_rank["ms_per_step"],
             "per_rank_gbs": per_rank["value"], "median_ms_per_step": per_rank["median_ms_per_step"],
             "clocks": {"sm_mhz": None, "reasons": [], "samples": 0}, "single_launch": per_rank["single_launch"]}
        nbytes, launches, kernel = text.size, 1, "k_scan_tma (one launch per step)"
        cfgd = {"workload": CONFIG_NAMES[cfg], "bytes_per_step": int(nbytes), "api": "sfa_match_async",
                "l2": "input > 126 MB L2: no flush needed" if nbytes > (126 << 20) else "input smaller than L2",
                "residency": per_rank["residency"], "parallelism": f"replicas x{world}"}
        wl = text

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    clocks = h["clocks"]
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    line = {
        "metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "median_ms_per_step": h["median_ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded, DESIGN.md input recipe)", "config": cfgd,
        "roofline": roofline(h["per_rank_gbs"], peak, peak_kind, nsm, sm_mhz, kernel,
                             ncu_traffic(f"cfg{cfg}"), int(nbytes), f"cfg{cfg}"),
        "clocks": clocks, "gpu_launches": launches * args.steps,
    }
    for k in ("single_launch", "uniform_api"):
        if k in h:
            line[k] = h[k]
    line["e2e"] = h.get("e2e")
    if cfg != 5:
        sfa = P.SFA(rx, alpha)
        pinned = torch.from_numpy(wl).pin_memory()
        sfa.match_host(pinned, stream)
        t0 = time.perf_counter()
        for _ in range(max(1, args.e2e_steps)):
            sfa.match_host(pinned, stream)
        e2e_s = (time.perf_counter() - t0) / max(1, args.e2e_steps)
        line["e2e"] = {"value": world * wl.size / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(wl.size),
                       "d2h_bytes_per_step": 8, "api": "sfa_match_host (pinned host text, sliced pipeline)"
                       + (f"; rank 0's replica alone, times {world} replicas" if world > 1 else "")}
        sfa.close()
    pcs = [int(c) for c in args.per_config.split(",") if c.strip()] if args.per_config else []
    per = {}
    for c in pcs:
        if c != cfg:
            per[f"cfg{c}"] = single_text_config(torch, P, c, stream, min(args.steps, 100) if c != 1 else 200,
                                                args.warmup, args.single_reps, peak, peak_kind, nsm, sm_mhz,
                                                spec=args.spec)
    if args.nsfa:
        per["ex3_n11"] = nsfa_compare(torch, P, stream, min(args.steps, 100), args.warmup, args.single_reps, peak,
                                      peak_kind, nsm, sm_mhz)
    if per:
        line["per_config"] = per
    if args.rn:
        line["rn_family"] = rn_family(torch, P, stream, args.warmup, peak, args.rn_bytes)
    if args.lazy:
        line["per_config"] = line.get("per_config", {})
        line["per_config"]["on_the_fly_r500_ra"] = lazy_family(torch, P, stream, args.warmup, peak, args.rn_bytes)
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_sample(cfg, rx, alpha, wl, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
