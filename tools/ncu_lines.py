"""Aggregate an ncu source page (cuda,sass CSV) per CUDA source line: instructions and stall samples."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file = cur_line = None
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    srcs = {}
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "Function Name" or hdr is None:
            continue
        if r[0] and r[0].isdigit():
            cur_line = (cur_file, int(r[0]))
            srcs[cur_line] = r[1]
            continue
        try:
            c = float(r[7] or 0)
            s = float(r[4] or 0)
        except (ValueError, IndexError):
            continue
        agg[cur_line][0] += c
        agg[cur_line][1] += s
    tot = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-instructions {tot:.4g}, stall samples {ts:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(top)]:
        if k is None:
            continue
        print(f"{k[0]}:{k[1]:4d} inst {v[0] / tot * 100:5.1f}%  smp {v[1] / ts * 100:5.1f}%  {srcs.get(k, '')[:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
