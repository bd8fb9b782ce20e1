"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv).

    python bench/launch_summary.py gpurun_out/launches.csv [title]
"""
import csv
import sys
from collections import defaultdict


def main(path, title=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iid = hdr.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        try:
            val = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        per[r[iid]][r[im]] = val
        names[r[iid]] = r[ik]
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    if title:
        print(title)
    print("share  launches  avg  dram-throughput  kernel")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{100 * t / tot:5.1f}%  {n:5d}  {t / n / 1e3:9.1f}us  {b / t if t else 0:8.0f} GB/s  {k[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
