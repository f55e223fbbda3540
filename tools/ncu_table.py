"""Summarise an ncu --set full report: one line per profiled launch."""
import csv
import subprocess
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_hit", "lts__t_sector_hit_rate.pct"),
    ("l1_hit", "l1tex__t_sector_hit_rate.pct"),
    ("warps_act", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("smem_dyn", "launch__shared_mem_per_block_dynamic"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    name_i = hdr.index("Kernel Name")
    print("kernel | " + " | ".join(m[0] for m in METRICS))
    for d in data:
        vals = []
        for label, m in METRICS:
            if m not in hdr:
                vals.append("NA")
                continue
            i = hdr.index(m)
            v = d[i].replace(",", "")
            u = units[i]
            try:
                f = float(v)
                if u == "byte":
                    f /= 1e6
                elif u == "Kbyte":
                    f /= 1e3
                elif u == "Gbyte":
                    f *= 1e3
                elif u == "msecond":
                    f *= 1e3
                elif u == "nsecond":
                    f /= 1e3
                vals.append(f"{f:.1f}")
            except ValueError:
                vals.append(v)
        print(d[name_i][:60] + " | " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
