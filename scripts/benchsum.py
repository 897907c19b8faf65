"""Print value / ms_per_step / roofline frac (and workload) of bench.py JSON lines.
Usage: python scripts/benchsum.py LOG..."""
import json
import sys

for f in sys.argv[1:]:
    line = None
    for ln in open(f, errors="replace"):
        if ln.startswith("{"):
            line = ln
    if line is None:
        print(f"{f}: no JSON line")
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    print(f"{f}: value={d.get('value'):.6g} {d.get('unit')} ms/step={d.get('ms_per_step'):.5g} "
          f"frac={r.get('frac')} launch_ms={r.get('avg_launch_ms')}")
