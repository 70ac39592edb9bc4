"""Per-source-line shared-memory wavefronts (actual / ideal / excessive) of a
kernel in an ncu report: where the L1/MIO time goes.

  python scripts/ncu_smem.py REPORT.ncu-rep [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
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
        if hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
            g = lambda name: float(r[hdr.index(name)] or 0) if r[hdr.index(name)] not in ("-", "") else 0.0
            agg.append((g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Ideal"), g("L2 Theoretical Sectors Global"),
                        fname, int(r[0]), r[1].strip()[:80]))
    tot = sum(a[0] for a in agg) or 1
    agg.sort(reverse=True)
    print(f"total shared wavefronts {tot:.4g}")
    for w, ideal, l2, f, ln, src in agg[:top]:
        print(f"{100.0 * w / tot:5.1f}% {f}:{ln:<4} wf={w:.3g} ideal={ideal:.3g} l2sect={l2:.3g} {src}")


if __name__ == "__main__":
    main()
