"""Compact table of an ncu --csv launch list (one row per kernel launch ≥ min_us)."""
import csv
import sys


def main(path, min_us=50.0):
    rows = list(csv.reader([l for l in open(path) if not l.startswith("==")]))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = {}
    for r in rows[1:]:
        d.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = r[vi].replace(",", "")
    for (i, k), m in sorted(d.items()):
        t = float(m.get("gpu__time_duration.sum", "0")) / 1e3
        if t < min_us:
            continue
        extra = " ".join(f"{n.split('__')[1][:22]}={float(v):.4g}" for n, v in m.items()
                         if n != "gpu__time_duration.sum")
        print(f"{i:4d} {t:10.1f} us  {k[:60]:60s} {extra}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 50.0)
