"""Per-kernel table from an ncu --metrics CSV of tools/nvlink_profile.py
(duration, DRAM, NVLink rx/tx per launch and device).

    python tools/ncu_nvl.py <csv> [kernel-substring]
"""
import collections
import csv
import sys


def rows(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    r = list(csv.reader(lines))
    hdr, body = r[0], r[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    k = collections.OrderedDict()
    for x in body:
        key = (int(x[ix["ID"]]), x[ix["Kernel Name"]].split("(")[0].replace("void ", ""),
               x[ix["Device"]])
        k.setdefault(key, {})[x[ix["Metric Name"]]] = float(x[ix["Metric Value"]].replace(",", ""))
    return k


def main():
    k = rows(sys.argv[1])
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    print("| id | kernel | dev | us | DRAM rd MB | DRAM wr MB | NVL rx MB | NVL tx MB | "
          "NVL rx GB/s | NVL tx GB/s | DRAM GB/s | warps active % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for (i, name, dev), m in k.items():
        if sub not in name:
            continue
        us = m.get("gpu__time_duration.sum", 0) / 1e3
        rd, wr = m.get("dram__bytes_read.sum", 0) / 1e6, m.get("dram__bytes_write.sum", 0) / 1e6
        rx, tx = m.get("nvlrx__bytes.sum", 0) / 1e6, m.get("nvltx__bytes.sum", 0) / 1e6
        gb = lambda mb: mb * 1e6 / (us * 1e-6) / 1e9 if us else 0.0
        print(f"| {i} | {name} | {dev} | {us:.1f} | {rd:.1f} | {wr:.1f} | {rx:.1f} | {tx:.1f} | "
              f"{gb(rx):.0f} | {gb(tx):.0f} | {gb(rd + wr):.0f} | "
              f"{m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} |")


if __name__ == "__main__":
    main()
