"""Digest of ncu --set full reports: duration, DRAM traffic, occupancy, top stalls."""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active%",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_sector_hit_rate.pct": "l2_hit%",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
}


def digest(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    stalls = []
    for h, u, v in zip(hdr, units, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if h in WANT:
            if u in ("nsecond", "ns") and WANT[h] == "us":
                x *= 1e-3
            if u in ("usecond",) and WANT[h] == "us":
                pass
            if u == "Kbyte":
                x *= 1e3
            if u == "Mbyte":
                x *= 1e6
            if u == "Gbyte":
                x *= 1e9
            d[WANT[h]] = x
        if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
            stalls.append((x, h.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", "")))
    stalls.sort(reverse=True)
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else path
    return name, d, stalls[:4]


if __name__ == "__main__":
    for p in sys.argv[1:]:
        name, d, st = digest(p)
        print(f"{name[:60]}: " + " ".join(f"{k}={v:.4g}" for k, v in d.items()) +
              " | stalls " + ", ".join(f"{n} {x:.1f}" for x, n in st))
