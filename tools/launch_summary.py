#!/usr/bin/env python
"""Per-kernel shares of an ncu launch list:
    ncu --metrics gpu__time_duration.sum --clock-control none -c N --csv --log-file launches.csv <command>
    python tools/launch_summary.py launches.csv "<command>" > profiles/rNN_bench_launches_summary.txt
(per-launch times under ncu are cold-cache and serialised: compare shares, not absolutes)."""
import collections
import csv
import re
import sys


def main():
    path, cmd = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
    rows = [r for r in csv.reader(l for l in open(path, errors="replace") if not l.startswith("=="))]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= iv or "gpu__time_duration" not in ",".join(r):
            continue
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1e-6)
        name = re.sub(r"\(.*", "", r[ik])
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    lev = sum(v for k, v in tot.items() if "lev_kernel" in k)
    nw = sum(v for k, v in tot.items() if "nw_" in k)
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none: {cmd}")
    print(f"# {sum(cnt.values())} launches, {total:.1f} ms total (cold-cache, serialised: compare shares); "
          f"lev_kernel (all buckets/sources) {100 * lev / total:.1f} %, NW kernels {100 * nw / total:.1f} %")
    for k, v in tot.most_common():
        print(f"{v:10.3f} ms {100 * v / total:6.2f} % {cnt[k]:6d} launches  {k}")


if __name__ == "__main__":
    main()
