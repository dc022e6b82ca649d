"""Per-source-line warp-stall samples and executed instructions from an ncu report
(needs -lineinfo builds), plus an executed-instruction breakdown by SASS opcode.

    python scripts/ncu_lines.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    func, path, hdr, agg, ops = "", "", None, {}, {}
    for r in rows:
        if len(r) == 2 and r[0] == "Function Name":
            func = r[1]
            continue
        if len(r) == 2 and r[0] == "File Path":
            path = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or kern not in func or not r:
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        if r[0] == "" and r[2].startswith("0x"):  # SASS row
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[3])
            if m:
                op = m.group(2)
                if op in ("LDG", "STG", "LD", "ST", "ATOM", "RED"):
                    op += (m.group(3) or "")[:12]
                ops[op] = ops.get(op, 0) + inst
            continue
        if r[0] in ("", "0"):
            continue
        key = (path.split("/")[-1], int(r[0]), r[1].strip()[:90])
        s, i = agg.get(key, (0, 0))
        agg[key] = (s + samples, i + inst)
    tot = sum(v[0] for v in agg.values()) or 1
    toti = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot}, warp instructions {toti}")
    print(" stall%  inst%  line")
    for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100.0 * v[0] / tot:6.1f} {100.0 * v[1] / toti:6.1f}  {f}:{ln:<5d} {src}")
    print("\nby instructions:")
    for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{100.0 * v[0] / tot:6.1f} {100.0 * v[1] / toti:6.1f}  {f}:{ln:<5d} {src}")
    print("\nby opcode:")
    toto = sum(ops.values()) or 1
    for op, v in sorted(ops.items(), key=lambda x: -x[1])[:top]:
        print(f"{100.0 * v / toto:6.1f}  {v:>10d}  {op}")


if __name__ == "__main__":
    main()
