"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import re
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    out = []
    for r in rows[1:]:
        name = r[ki]
        name = re.sub(r"\(.*$", "", name)
        name = name.replace("ds::<unnamed>::", "").replace("ds::", "")
        name = re.sub(r"^void ", "", name)
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
        out.append((name, v * scale.get(r[ui], 1.0)))
    return out


def main(path, skip=0, top=40):
    rows = load(path)[skip:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, us in rows:
        agg[n][0] += 1
        agg[n][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"launches {len(rows)}  total {tot / 1e3:.3f} ms (serialised, cold-cache)")
    print(f"{'kernel':56s} {'launches':>8s} {'total_us':>10s} {'us/launch':>9s} {'share':>6s}")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{n[:56]:56s} {c:8d} {t:10.1f} {t / c:9.2f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
