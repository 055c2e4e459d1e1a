"""Per-CUDA-line instruction counts and stall samples from an .ncu-rep (cuda,sass view)."""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    i_exe, i_st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows[hi + 1:]:
        if len(r) <= i_exe or r[2] != "-":
            continue  # keep only the per-CUDA-line aggregate rows
        try:
            lines.append((int(r[0]), r[1], float(r[i_exe] or 0), float(r[i_st] or 0)))
        except ValueError:
            continue
    te = sum(x[2] for x in lines) or 1
    ts = sum(x[3] for x in lines) or 1
    print(f"total warp-instructions {te:.3e}")
    for ln, src, e, s in sorted(lines, key=lambda x: -x[2])[:top]:
        print(f"{ln:5d} inst {100 * e / te:5.1f}%  stall {100 * s / ts:5.1f}%  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
