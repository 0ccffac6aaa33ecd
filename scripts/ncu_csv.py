"""Print an ncu --csv metrics log as one row per launch (kernel, metric values)."""
import csv
import io
import sys
from collections import OrderedDict


def load(path):
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ii, ki, mi, vi = (hdr.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    out = OrderedDict()
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        d = out.setdefault(r[ii], {"kernel": r[ki]})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            d[r[mi]] = r[vi]
    return list(out.values())


if __name__ == "__main__":
    for i, d in enumerate(load(sys.argv[1])):
        k = d.pop("kernel")
        print(i, k[:60])
        for m, v in d.items():
            print(f"    {m:70s} {v}")
