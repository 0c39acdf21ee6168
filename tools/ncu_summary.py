"""Summarise ncu outputs into profiles/ (run in the build container).

    python tools/ncu_summary.py launches <launches.csv> <out.md>
    python tools/ncu_summary.py report <prof.ncu-rep> <out.md> [algorithmic_bytes]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__waves_per_multiprocessor",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__maximum_warps_per_active_cycle_pct", "lts__t_sector_hit_rate.pct",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio"]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[4]
        short = name.split("(")[0][:90] if "dsgd" in name else name.split("(")[0].split("<")[0][:60]
        agg[short][0] += 1
        agg[short][1] += float(r[-1]) / 1e3
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list: {path}\n\n`ncu --metrics gpu__time_duration.sum "
                f"--clock-control none` (cold-cache, serialised: compare shares)\n\n")
        f.write("| launches | total us | share | kernel |\n|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | `{k}` |\n")
    print(open(out).read())


def report(path, out, alg_bytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: {path}\n\n")
        for vals in rows[2:]:
            kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            f.write(f"## `{kname[:120]}`\n\n| metric | value | unit |\n|---|---|---|\n")
            m = {}
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    m[k] = (vals[i], units[i])
                    f.write(f"| {k} | {vals[i]} | {units[i]} |\n")
            if alg_bytes and "dram__bytes_read.sum" in m:
                def mb(v):
                    x, u = float(v[0].replace(",", "")), v[1]
                    return x * {"Gbyte": 1e3, "Mbyte": 1, "Kbyte": 1e-3, "byte": 1e-6}.get(u, 1)
                traffic = mb(m["dram__bytes_read.sum"]) + mb(m["dram__bytes_write.sum"])
                f.write(f"\nDRAM traffic {traffic:.1f} MB vs algorithmic {alg_bytes / 1e6:.1f} MB "
                        f"(ratio {traffic / (alg_bytes / 1e6):.3f}; writes still dirty in L2 at "
                        f"kernel end are not counted)\n\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        report(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
