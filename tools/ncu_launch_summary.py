"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys


def summarise(path, header_lines=()):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        agg[r[ki][:110]][0] += 1
        agg[r[ki][:110]][1] += v
    tot = sum(v[1] for v in agg.values())
    out = list(header_lines) + ["# launches  total_us  share  avg_us  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{v[0]:5d} {v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}% {v[1] / 1e3 / v[0]:8.2f}  {k}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print(summarise(sys.argv[1], ["# " + " ".join(sys.argv[2:])] if len(sys.argv) > 2 else []), end="")
