"""Aggregate ncu warp-stall samples per CUDA source line from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`.
Usage: python scripts/ncu_source_stalls.py file.csv [top]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    agg, cur_file, cur = {}, None, None
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:
            cur = (cur_file, int(r[0]), r[1].strip()[:90])
            agg.setdefault(cur, 0)
            try:
                agg[cur] += int(r[4])
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    print(f"# {tot} warp-stall samples")
    for (f, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
