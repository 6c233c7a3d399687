"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
count, total and share of device time (cold-cache, serialised: compare shares)."""
import csv
import re
import sys
from collections import defaultdict


def main(path, per_call=None):
    """per_call: number of run_distributed calls captured; kernels launched at least
    that many times are the per-step ones (setup kernels -- graph generation, world
    build -- appear once and are listed separately)."""
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("(anonymous namespace)::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
        ms = v * scale.get(unit, 1e-6)
        tot[name] += ms
        cnt[name] += 1
    keys = [k for k in tot if per_call is None or cnt[k] >= per_call]
    T = sum(tot[k] for k in keys)
    hdr = "per-step kernels" if per_call else "all kernels"
    print(f"{hdr:60s} {'launches':>8s} {'total ms':>10s} {'avg us':>9s} {'share':>7s}")
    for k in sorted(keys, key=lambda x: -tot[x]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.3f} {1e3 * tot[k] / cnt[k]:9.1f} {100 * tot[k] / T:6.1f}%")
    print(f"{'TOTAL':60s} {sum(cnt[k] for k in keys):8d} {T:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
