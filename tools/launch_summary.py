"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launch
count, total and mean device time, and share of the timed step (the last `--steps` steps:
everything after the last warm-up step's final espo kernel is hard to delimit, so the
summary reports shares over all espo kernels of the run and over one steady-state step,
i.e. the launches between the last two `k_prepare_groups` launches)."""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    m = re.search(r"(k_[a-z_]+)(<[^(]*>)?", name)
    if m:
        return m.group(1) + (m.group(2) or "")
    return name.split("(")[0][:60]


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        rows.append((short(r["Kernel Name"]), ns))
    return rows


def table(rows, title):
    agg = OrderedDict()
    for k, ns in rows:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values())
    out = [f"### {title}", "", "| kernel | launches | total ms | mean µs | share |", "|---|---|---|---|---|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | {ns / tot * 100:.1f}% |")
    out.append(f"| total | {sum(a[0] for a in agg.values())} | {tot / 1e6:.3f} | | 100% |")
    return "\n".join(out)


def main(path):
    rows = [r for r in load(path)]
    espo = [r for r in rows if r[0].startswith("k_")]
    idx = [i for i, r in enumerate(espo) if r[0].startswith("k_prepare_groups")]
    print(table(espo, "all libespo launches of the run (warm-up + timed)"))
    if len(idx) >= 1:
        step = espo[idx[-1]:]
        print()
        print(table(step, "one steady-state step (launches from the last k_prepare_groups)"))


if __name__ == "__main__":
    main(sys.argv[1])
