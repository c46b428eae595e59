"""Condensed table of an `ncu -i rep --page raw --csv` export: one column per
captured launch, the rows the NTT analysis in DESIGN.md uses.
python tools/ncu_raw_table.py file.csv [...]"""
import csv
import re
import sys

ROWS = [
    ("gpu__time_duration (us)", "gpu__time_duration.sum"),
    ("registers / thread", "launch__registers_per_thread"),
    ("warps active (% of peak)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("warp instructions executed (M)", "smsp__inst_executed.sum"),
    ("FP64 pipe (% active)", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("ALU pipe (% active)", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("FMA-heavy pipe (% elapsed)", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("issue active (%)", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("l1tex throughput (%)", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("L2 hit rate (%)", "lts__t_sector_hit_rate.pct"),
    ("DRAM throughput (%)", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("DRAM read (MB)", "dram__bytes_read.sum"),
    ("DRAM write (MB)", "dram__bytes_write.sum"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    names = []
    for r in data:
        m = re.search(r"k_ntt_phase<([^>]*)>", r[col["Kernel Name"]])
        names.append("<" + m.group(1).replace(" ", "") + ">" if m else r[col["Kernel Name"]][:24])
    print(path)
    print(f"{'':34s}| " + " | ".join(f"{n:>14s}" for n in names))
    for label, key in ROWS:
        if key not in col:
            continue
        vals = []
        for r in data:
            v = r[col[key]].replace(",", "")
            try:
                f = float(v)
                u = units[col[key]]
                if key.endswith("inst_executed.sum"):
                    f /= 1e6
                elif "bytes" in key:
                    f = f / 1e6 if u == "byte" else f * {"Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
                elif key.startswith("gpu__time") and u in ("ns", "nsecond"):
                    f /= 1e3
                vals.append(f"{f:14.1f}")
            except ValueError:
                vals.append(f"{v:>14s}")
        print(f"{label:34s}| " + " | ".join(vals))
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio")
             or h.startswith("smsp__average_warp_latency_issue_stalled")]
    if stall:
        tops = []
        for r in data:
            s = sorted(((float(r[col[h]].replace(",", "") or 0), h) for h in stall), reverse=True)[:3]
            tops.append(", ".join(f"{re.sub(r'.*stalled_|_per_issue.*|.ratio', '', h)} {v:.1f}" for v, h in s))
        for n, t in zip(names, tops):
            print(f"top stalls {n}: {t}")
    print()


for p in sys.argv[1:]:
    main(p)
