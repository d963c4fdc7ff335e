"""Top SASS lines by warp-stall samples from an ncu report (source page).

    python tools/ncu_hot.py report.ncu-rep [N] [--kernel SUBSTR]
"""
import csv
import io
import subprocess
import sys


def main() -> None:
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
    kern = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if kern and kern not in name:
            continue
        rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
        h = rows[0]
        iS, iA = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        body = [r for r in rows[1:] if len(r) > iA and r[iA].isdigit()]
        tot = sum(int(r[iA]) for r in body)
        print(name[:120], "total samples", tot)
        # aggregate by opcode too
        ops = {}
        for r in body:
            op = r[iS].strip().split()[0] if r[iS].strip() else "?"
            if op.startswith("@"):
                op = r[iS].strip().split()[1]
            ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + int(r[iA])
        print("by opcode:", sorted(ops.items(), key=lambda kv: -kv[1])[:15])
        for r in sorted(body, key=lambda r: -int(r[iA]))[:n]:
            print(f"{int(r[iA]):6d} {r[0]} {r[iS].strip()[:90]}")


if __name__ == "__main__":
    main()
