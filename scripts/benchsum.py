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
    nv = d.get("nvlink") or {}
    extra = ""
    if nv:
        extra = (f" zsync_ms={nv.get('fused_zsync_ms') or 0:.4f} rs_ms={nv.get('reduce_scatter_ms') or 0:.4f}"
                 f" ag_ms={nv.get('all_gather_ms') or 0:.4f}")
    fr = r.get("frac")
    print(f"{f}: value={d.get('value'):.6g} {d.get('unit')} ms/step={d.get('ms_per_step'):.5g} "
          f"frac={fr if fr is None else round(fr, 4)} launch_ms={r.get('avg_launch_ms')}{extra}")
