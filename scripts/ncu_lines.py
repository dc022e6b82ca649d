"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo builds).

    python scripts/ncu_lines.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    func, path, hdr, agg = "", "", None, {}
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
        if not hdr or kern not in func or not r or r[0] in ("", "0"):
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        key = (path.split("/")[-1], int(r[0]), r[1].strip()[:90])
        agg[key] = agg.get(key, 0) + samples
    tot = sum(agg.values()) or 1
    print(f"total samples {tot}")
    for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{100.0 * v / tot:5.1f}%  {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main()
