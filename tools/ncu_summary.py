"""Key counters per captured launch from `ncu -i X.ncu-rep --page raw --csv` output.

usage: python tools/ncu_summary.py gpurun_out/r02_extend_add_raw.csv [...]
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64act_%"),
    ("lts__t_sector_hit_rate.pct", "l2hit_%"),
]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def main():
    for path in sys.argv[1:]:
        with open(path) as f:
            rows = list(csv.reader(l for l in f if not l.startswith("==")))
        if len(rows) < 3:
            print(path, ": no launches")
            continue
        hdr, units = rows[0], rows[1]
        col = {h: i for i, h in enumerate(hdr)}
        print("##", path)
        for r in rows[2:]:
            if len(r) < len(hdr):
                continue
            name = r[col["Kernel Name"]].split("(")[0][-48:]
            grid = r[col.get("Grid Size", 0)]
            out = ["%-48s grid %-14s" % (name, grid)]
            for k, lab in KEYS:
                if k in col:
                    v = num(r[col[k]])
                    u = units[col[k]]
                    if v is None:
                        continue
                    if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                        v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u]
                        out.append("%s %.2f MB" % (lab, v))
                    elif u in ("ns", "us", "ms", "nsecond", "usecond", "msecond"):
                        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}[u]
                        out.append("%s %.1f us" % (lab, v))
                    else:
                        out.append("%s %.1f" % (lab, v))
            print("  ".join(out))


if __name__ == "__main__":
    main()
