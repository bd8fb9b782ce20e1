"""Aggregate ncu 'Instructions Executed' per CUDA source line from a
`--print-source cuda,sass` CSV dump (usage: lineprof.py dump.csv [top])."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
per = collections.Counter()
src = {}
cur = cur_file = None
total = 0.0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        try:
            cur = (cur_file, int(r[0]))
            src[cur] = r[1][:95]
        except ValueError:
            pass
        continue
    if len(r) > 7 and r[2].startswith("0x"):
        try:
            ex = float(r[7].replace(",", ""))
        except ValueError:
            continue
        per[cur] += ex
        total += ex
print("total warp-instructions", total)
for k, c in per.most_common(top):
    print(f"{c / total * 100:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')}")
