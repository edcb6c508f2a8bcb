"""Per-launch table of an ncu --csv --metrics launch list: id, kernel, metrics (development aid)."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = OrderedDict()
    for r in rows[hdr + 1:]:
        d.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = r[vi].replace(",", "")
    return d


if __name__ == "__main__":
    d = load(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    for (i, k), v in list(d.items())[:n]:
        print(i, k.split("(")[0][:40], " ".join(f"{m.split('.')[0].split('__')[-1]}={x}" for m, x in v.items()))
