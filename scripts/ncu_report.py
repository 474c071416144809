"""Markdown summary rows from ncu --set full reports (one row per captured launch)."""
import csv
import io
import re
import subprocess
import sys

M = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "DRAM rd"),
     ("dram__bytes_write.sum", "DRAM wr"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
     ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
     ("launch__block_size", "block"), ("lts__t_sector_hit_rate.pct", "L2 hit %"),
     ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb")]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    h, units = r[0], r[1]
    res = []
    for v in r[2:]:
        name = re.sub(r"\(.*", "", v[h.index("Kernel Name")]).split("::")[-1]
        vals = []
        for key, _ in M:
            if key in h:
                i = h.index(key)
                u = units[i]
                vals.append(f"{v[i]} {u}".strip() if u in ("Mbyte", "Kbyte", "Gbyte", "byte") else v[i])
            else:
                vals.append("")
        res.append([name] + vals)
    return res


def main(paths):
    print("| kernel | " + " | ".join(n for _, n in M) + " |")
    print("|---" * (len(M) + 1) + "|")
    for p in paths:
        for r in rows(p):
            print("| " + " | ".join(r) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
