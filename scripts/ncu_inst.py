"""Per-source-line executed warp instructions of one kernel in an ncu report,
grouped, with the share of the kernel total.

  python scripts/ncu_inst.py REPORT.ncu-rep [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, fname, agg = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) > 7 and r[0].isdigit() and r[2] == "-":
            ex = int(r[7]) if r[7] not in ("-", "") else 0
            agg.append((ex, fname, int(r[0]), r[1].strip()[:90]))
    tot = sum(a[0] for a in agg) or 1
    agg.sort(reverse=True)
    print(f"total warp instructions {tot:.4g}")
    for ex, f, ln, src in agg[:top]:
        print(f"{100.0 * ex / tot:5.1f}% {f}:{ln:<4} {ex:>11} {src}")


if __name__ == "__main__":
    main()
