"""Markdown table of an end-of-round evidence directory: python scripts/eor_table.py profiles/r01_vNN"""
import glob
import json
import os
import sys

d = sys.argv[1]
print("| run | value (utt/s) | ms/step | roofline (dominant kernel) | e2e | cpu_baseline |")
print("|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
    name = os.path.basename(f)[6:-5]
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    if name == "reference":
        print(f"| `reference` (`--impl reference`, the CPU oracle) | {j['value']:,.2f} | {j['ms_per_step']:.1f} | — | — "
              f"| {j['cpu_baseline']['cores']} cores |")
        continue
    r = j["roofline"]
    e2e = j.get("e2e") or {}
    cpu = j.get("cpu_baseline") or {}
    ach = f"{r['achieved']:,.0f} {r['unit']} ({r['frac']:.3f} of {r['peak']})"
    print(f"| `{name}` | {j['value']:,.1f} | {j['ms_per_step']:.3f} | {r['kernel']} {ach} | "
          f"{e2e.get('value') and round(e2e['value'], 1)} | {cpu.get('value') and round(cpu['value'], 2)} |")
