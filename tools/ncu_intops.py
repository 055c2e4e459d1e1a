"""Per-CUDA-line SASS opcode mix from an .ncu-rep (cuda,sass view): which
source lines issue the integer/control overhead."""
import collections
import csv
import io
import subprocess
import sys

INT = {'IMAD', 'ISETP', 'LOP3', 'BRA', 'VIADD', 'LEA', 'SHF', 'IADD3', 'SEL', 'PLOP3', 'BSSY', 'BSYNC', 'R2UR', 'NOP',
       'LDCU', 'IABS', 'I2F', 'F2I', 'UMOV', 'ULEA', 'S2UR', 'WARPSYNC', 'YIELD', 'LDC', 'MOV', 'SHL', 'IMNMX',
       'VIMNMX', 'FSEL', 'P2R', 'R2P', 'UIADD3', 'ULOP3', 'USHF', 'UISETP', 'I2FP', 'F2IP'}


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    per = collections.defaultdict(collections.Counter)
    src = {}
    fname, cur, iex = "?", None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "Line No":
            iex = r.index("Instructions Executed")
            continue
        if r[0] and not r[0].isdigit():
            fname = r[-1] if len(r) > 1 else r[0]
            continue
        if r[0]:
            cur = (fname.split("/")[-1], int(r[0]))
            src[cur] = r[1]
            continue
        if iex is None or cur is None:
            continue
        try:
            n = float(r[iex] or 0)
        except ValueError:
            continue
        s = r[3].split()
        if not s:
            continue
        op = s[1] if s[0].startswith('@') else s[0]
        per[cur][op.split('.')[0]] += n
    tot = sum(sum(c.values()) for c in per.values()) or 1
    intl = sorted(((sum(v for k, v in c.items() if k in INT), ln) for ln, c in per.items()), reverse=True)
    print("warp-instructions %.3e, integer/control share %.1f%%" % (tot, 100 * sum(x for x, _ in intl) / tot))
    for x, ln in intl[:top]:
        c = per[ln]
        print(f"{ln[0][:10]:10s}{ln[1]:5d} {100 * x / tot:5.1f}% {src[ln].strip()[:60]:60s} {dict(c.most_common(4))}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
