"""Summarise an ncu report (``ncu --set full`` capture of one k_scan_tma launch)
into profiles/ncu_summary.json under a config key; bench.py reads the DRAM
traffic per launch from there (roofline.traffic).

    python scripts/ncu_summary.py <report.ncu-rep | raw.csv> <cfgN> [note]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_pct_peak": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1e-9),
    "smem_wavefronts_ld": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 1),
    "smem_bank_conflicts_ld": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1),
    "smem_wavefronts_pct_peak": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warp_inst": ("smsp__inst_executed.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
              "msecond": 1e6, "ms": 1e6, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def main():
    rep, key = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    if rep.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` output, exported on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")], "report": os.path.basename(rep), "note": note}
    for name, (metric, scale) in KEYS.items():
        if metric not in hdr:
            continue
        i = hdr.index(metric)
        v = float(vals[i].replace(",", ""))
        v *= UNIT_SCALE.get(units[i], 1)
        if name == "duration_us":
            v = v / 1e3  # ns -> us
        elif name == "sm_clock_ghz":
            v = v / 1e9
        d[name] = v
    d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    allv = json.load(open(path)) if os.path.exists(path) else {}
    allv[key] = d
    json.dump(allv, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
