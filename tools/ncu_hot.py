"""Top SASS instructions by warp-stall samples from an ncu report (read here, no GPU).

    python tools/ncu_hot.py report.ncu-rep [N]
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    iex = hdr.index("Instructions Executed")
    body = rows[2:]
    tot = sum(float(r[isamp] or 0) for r in body)
    idx = {r[ia]: i for i, r in enumerate(body)}
    print(f"{rows[0][1]}\n total samples {tot:.0f}, {len(body)} instructions")
    top = sorted(body, key=lambda r: -float(r[isamp] or 0))[:n]
    for r in top:
        i = idx[r[ia]]
        print(f"{i:5d} {float(r[isamp]) / tot:6.3f} ex={r[iex]:>9s}  {r[isrc].strip()[:90]}")


if __name__ == "__main__":
    main()
