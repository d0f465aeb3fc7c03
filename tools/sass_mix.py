"""Executed SASS opcode mix of an ncu source-page CSV (ncu -i X --page source --csv --print-source
sass): warp-instructions per opcode, most frequent first, and the total."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    out = collections.defaultdict(collections.Counter)
    kernel = None
    hdr = None
    for r in rows:
        if r and r[0] == "Kernel Name":
            kernel = r[1][:80]
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            n = int(d["Instructions Executed"])
        except (KeyError, ValueError):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9]+)(\.[A-Z0-9_.]+)?", d["Source"].strip())
        op = m.group(2) if m else "?"
        if op in ("IMAD", "MUFU"):
            op += m.group(3) or ""
        out[kernel][op] += n
    for k, c in out.items():
        tot = sum(c.values())
        print(f"{k}: {tot} warp-instructions")
        print("  " + " ".join(f"{op}:{n / tot * 100:.1f}%" for op, n in c.most_common(25)))


if __name__ == "__main__":
    main(sys.argv[1])
