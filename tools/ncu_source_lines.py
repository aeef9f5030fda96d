"""Per-CUDA-source-line share of warp-stall samples and executed instructions
from `ncu -i REP --page source --csv --print-source cuda,sass`.

    python tools/ncu_source_lines.py SOURCE.csv [TOP]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    fp, hdr, out = None, None, []
    for r in csv.reader(open(path)):
        if len(r) == 2 and r[0] == "File Path":
            fp = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] and r[2] == "-":
            d = dict(zip(hdr, r))
            out.append((fp, int(r[0]), r[1].strip(),
                        float(d["Warp Stall Sampling (All Samples)"] or 0),
                        float(d["Instructions Executed"] or 0)))
    ts = sum(o[3] for o in out) or 1.0
    ti = sum(o[4] for o in out) or 1.0
    print(f"samples {ts:.0f}  warp instructions {ti:.0f}")
    for o in sorted(out, key=lambda o: -o[3])[:top]:
        print(f"{o[0][:24]:24s} {o[1]:4d}  stall {o[3] / ts:5.3f}  inst {o[4] / ti:5.3f}  {o[2][:90]}")


if __name__ == "__main__":
    main()
