"""Per-CUDA-source-line stall samples and executed instructions from an ncu report
(ncu --page source --print-source cuda,sass).  usage: ncu_lines.py <rep> [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, rows = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0].isdigit() and len(r) >= len(hdr):
            # ncu does not escape quotes inside source text: take the metrics from the right
            rows.append((cur, int(r[0]), r[1], r[len(r) - len(hdr):]))
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    ts = sum(f(r[3][si]) for r in rows) or 1
    ti = sum(f(r[3][ii]) for r in rows) or 1
    rows.sort(key=lambda r: -f(r[3][si]))
    for fn, ln, src, r in rows[:top]:
        print(f"{fn}:{ln:4d} samp {100 * f(r[si]) / ts:5.1f}% ins {100 * f(r[ii]) / ti:5.1f}%  {src.strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
