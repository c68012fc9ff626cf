"""Prints the headline and per-config GB/s of a bench line (default gpurun_out/q_bench.json)."""
import json
import sys

d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/q_bench.json").read().strip().splitlines()[-1])
print("cfg5", round(d["value"]), round(d["single_launch"]["gbs"]))
for k, v in d.get("per_config", {}).items():
    if "value" in v:
        print(k, round(v["value"]), round(v["single_launch"]["gbs"]))
