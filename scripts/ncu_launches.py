"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, mean / total duration and share of the listed time.

  python scripts/ncu_launches.py gpurun_out/launches_X.csv profiles/r01_launches_cfg2.txt [--skip REGEX]
"""
import csv
import re
import sys
from collections import OrderedDict


def main():
    src, dst = sys.argv[1], sys.argv[2]
    skip = re.compile(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else None
    rows = [r for r in csv.DictReader(l for l in open(src) if l.startswith('"'))]
    per = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").strip()
        name = re.sub(r"^.*unnamed>::", "", name)
        if skip and skip.search(name):
            continue
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1e-6)
        key = f"{name} grid{r['Grid Size']} block{r['Block Size']}"
        e = per.setdefault(key, [0, 0.0])
        e[0] += 1
        e[1] += v
    total = sum(v for _, v in per.values()) or 1.0
    lines = [f"source: {src}", "per-launch gpu__time_duration (ncu, --clock-control none, serialised, cold-ish caches)",
             f"{'kernel':78s} {'launches':>8s} {'mean ms':>10s} {'total ms':>10s} {'share':>7s}"]
    for k, (n, v) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:78]:78s} {n:8d} {v / n:10.4f} {v:10.3f} {100 * v / total:6.1f}%")
    lines.append(f"{'total':78s} {sum(n for n, _ in per.values()):8d} {'':>10s} {total:10.3f}")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
