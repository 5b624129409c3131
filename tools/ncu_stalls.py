"""Top warp-stall SASS lines of one ncu --set full capture, with context:
    python tools/ncu_stalls.py gpurun_out/x.ncu-rep [top=20] [context=0]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, rows = r[1], r[2:]
    i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    tot = sum(int(x[i_s] or 0) for x in rows)
    print("kernel:", r[0][1][:120], "| samples:", tot)
    order = sorted(range(len(rows)), key=lambda k: -int(rows[k][i_s] or 0))[:top]
    for k in order:
        for j in range(max(0, k - ctx), min(len(rows), k + 1)):
            x = rows[j]
            print(f"{x[i_s]:>6} {100.0 * int(x[i_s] or 0) / tot:5.1f}% {x[0][-5:]} {x[i_src][:90]}")
        if ctx:
            print("---")


if __name__ == "__main__":
    main()
