"""Aggregate an ncu --csv launch list (gpu__time_duration.sum and optional
metrics) by kernel name and grid: python tools/launches.py file.csv [top]"""
import csv
import collections
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, ni, vi, gi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Grid Size"), h.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        per[r[ii]][r[ni]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "") + " " + r[gi]
    return per, names


def main():
    per, names = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    tot = 0.0
    for i, m in per.items():
        k = names[i]
        cnt[k] += 1
        for mn, v in m.items():
            agg[k][mn] += v
        tot += m.get("gpu__time_duration.sum", 0.0)
    mets = sorted({mn for m in per.values() for mn in m} - {"gpu__time_duration.sum"})
    print(f"total {tot / 1e6:.3f} ms over {len(per)} launches")
    order = sorted(agg, key=lambda k: -agg[k]["gpu__time_duration.sum"])
    for k in order[:top]:
        t = agg[k]["gpu__time_duration.sum"]
        extra = []
        for mn in mets:
            v = agg[k][mn]
            if "pct" in mn:
                extra.append(f"{mn.split('.')[0].split('__')[-1]}={v / cnt[k]:.1f}%")
            else:
                extra.append(f"{mn.split('.')[0].split('__')[-1]}={v / cnt[k]:.3g}")
        print(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}% n={cnt[k]:4d} {k}  " + " ".join(extra))


def fine_window(path, regex, first, n):
    """The --launch-skip (counted over kernels matching regex) that starts an
    n-launch window at the longest `first` launch followed by n-1 matches."""
    import re
    per, names = load(path)
    ids = sorted(per, key=int)
    m = [i for i in ids if re.search(regex, names[i])]
    best, at = -1.0, 0
    for j, i in enumerate(m[:len(m) - n + 1]):
        if first in names[i]:
            t = sum(per[k].get("gpu__time_duration.sum", 0.0) for k in m[j:j + n])
            if t > best:
                best, at = t, j
    return at


if __name__ == "__main__":
    if sys.argv[1] == "--skip":
        print(fine_window(sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5])))
    else:
        main()
