"""Summarise an ncu --set full report into a markdown table (for profiles/).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--units kernel=count ...]

--units maps a kernel-name substring to the number of algorithmic units one
launch processed (queries / points / records) so DRAM bytes per unit can be
compared with the algorithmic bytes per unit of DESIGN.md.
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1TEX %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def load(path: str):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v: str, unit: str) -> float:
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v.replace(",", "")) * mult


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--units", nargs="*", default=[])
    args = ap.parse_args()
    units = dict(u.split("=") for u in args.units)
    hdr, unit_row, rows = load(args.report)
    cols = [(hdr.index(m), label) for m, label in METRICS if m in hdr]
    print("| kernel | " + " | ".join(label for _, label in cols) + " | DRAM B/unit |")
    print("|---" * (len(cols) + 2) + "|")
    for r in rows:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        cells = []
        for i, label in cols:
            v, u = r[i], unit_row[i]
            if "bytes" in hdr[i]:
                cells.append(f"{to_bytes(v, u) / 1e6:.1f} MB")
            elif hdr[i] == "gpu__time_duration.sum":
                cells.append(f"{float(v.replace(',', '')):.1f} {u}")
            else:
                cells.append(v)
        per = ""
        for key, n in units.items():
            if key in name:
                rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], unit_row[hdr.index("dram__bytes_read.sum")])
                wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], unit_row[hdr.index("dram__bytes_write.sum")])
                per = f"{(rd + wr) / float(n):.2f}"
        print(f"| {name} | " + " | ".join(cells) + f" | {per} |")


if __name__ == "__main__":
    main()
