"""Summarize an ncu report (raw page) into a small text table for profiles/."""
import csv, subprocess, sys

METRICS = [
    ("gpu__time_duration.sum", "us"), ("launch__grid_size", ""), ("launch__block_size", ""),
    ("launch__registers_per_thread", ""), ("launch__shared_mem_per_block_dynamic", "KB"),
    ("dram__bytes_read.sum", "MB"), ("dram__bytes_write.sum", "MB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    name_i = idx.get("Kernel Name")
    print(f"# ncu --set full summary of {rep}")
    for n, d in enumerate(rows[2:]):
        print(f"launch {n}: {d[name_i][:90] if name_i is not None else ''}")
        for m, _ in METRICS:
            if m in idx:
                print(f"    {m:70s} {d[idx[m]]:>14s} {units[idx[m]]}")


if __name__ == "__main__":
    main(sys.argv[1])
