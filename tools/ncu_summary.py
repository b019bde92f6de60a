"""Summarise an ncu --set full report (one kernel launch per line) as markdown.
usage: python tools/ncu_summary.py report.ncu-rep [title] > profiles/.../x.md"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "int8 tensor pipe active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe inst %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# {title}\n")
    print("| launch | kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 2) + "|")
    for n, r in enumerate(data):
        name = r[idx["Kernel Name"]].split("(")[0][-60:] if "Kernel Name" in idx else "?"
        vals = []
        for k, _ in KEYS:
            if k in idx:
                u = units[idx[k]]
                vals.append(f"{r[idx[k]]} {u}".strip())
            else:
                vals.append("n/a")
        print(f"| {n} | `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
