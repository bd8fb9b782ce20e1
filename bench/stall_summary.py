"""Warp-stall breakdown of one ncu --set full --import-source on capture (source page):

    python bench/stall_summary.py gpurun_out/prof.ncu-rep [cubin-with-lineinfo kernel-symbol-substring] > profiles/rNN_ncu_stalls.txt

Prints the stall reasons over the whole kernel and, when the object file is given, the source lines
(nvdisasm -g) that hold the most samples."""
import collections
import csv
import re
import subprocess
import sys


def main(rep, cubin=None, sym=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    print(rows[0][1])
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except ValueError:
            return 0.0

    def addr(r):
        a = r[ix["Address"]]
        return int(a, 16) if a.startswith("0x") else int(a)

    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(f(r, "# Samples") for r in data)
    print(f"warp samples: {tot:.0f}; warp instructions executed: {sum(f(r, 'Instructions Executed') for r in data):.4g}")
    agg = {s: sum(f(r, s) for r in data) for s in stalls}
    for s, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {s:26s} {100 * v / tot:5.1f}%")
    if not cubin:
        return
    txt = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(txt) if l.startswith(".text.") and sym in l][0]
    amap, cur = {}, None
    for l in txt[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,6})\*/", l)
        if m:
            amap[int(m.group(1), 16)] = cur
    base = min(addr(r) for r in data)
    by, top = collections.Counter(), collections.defaultdict(collections.Counter)
    for r in data:
        ln = amap.get(addr(r) - base)
        by[ln] += f(r, "# Samples")
        for s in stalls:
            top[ln][s] += f(r, s)
    print("source lines by samples (file, line, share, top stall):")
    for ln, v in by.most_common(25):
        t = top[ln].most_common(1)[0]
        print(f"  {str(ln):38s} {100 * v / tot:5.1f}%  {t[0]} {100 * t[1] / max(v, 1):.0f}%")


if __name__ == "__main__":
    main(*sys.argv[1:4])
