"""Summarise ncu captures into profiles/ (run here, after gpurun brought the .ncu-rep back).

    python bench/profile_summary.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv profiles/r01

Writes <prefix>_ncu_full.txt (key metrics of the top kernel), <prefix>_launches.csv
(copied launch list) and updates profiles/ncu_summary.json (per-launch DRAM
traffic used by bench.py's roofline.traffic)."""

import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]


def main(rep, launches, prefix):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = []
    summ_path = Path("profiles/ncu_summary.json")
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        rec = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = (vals[i], units[i])
        lines.append(f"kernel: {name}")
        for k, (v, u) in rec.items():
            lines.append(f"  {k} = {v} {u}")
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd = float(rec["dram__bytes_read.sum"][0].replace(",", "")) * scale.get(rec["dram__bytes_read.sum"][1], 1.0)
        wr = float(rec["dram__bytes_write.sum"][0].replace(",", "")) * scale.get(rec["dram__bytes_write.sum"][1], 1.0)
        t = float(rec["gpu__time_duration.sum"][0].replace(",", ""))
        tu = rec["gpu__time_duration.sum"][1]
        t_ms = t / 1e6 if tu == "ns" else (t / 1e3 if tu == "us" else t)
        key = "wtv_prox_kernel" if "wtv" in name else name.split("(")[0]
        summ[key] = {"kernel": name, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                     "ncu_time_ms": t_ms, "source": str(rep)}
    Path(prefix + "_ncu_full.txt").write_text("\n".join(lines) + "\n")
    summ_path.write_text(json.dumps(summ, indent=1) + "\n")
    if launches and Path(launches).exists():
        shutil.copy(launches, prefix + "_launches.csv")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "profiles/r01")
