"""Per-source-line summary of an ncu report (instructions executed, stall
samples), from `ncu -i REP --page source --csv --print-source cuda,sass`.

    python tools/ncu_lines.py REP.ncu-rep [top]
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
    rows = []
    fname = "?"
    hdr = None
    for line in out.splitlines():
        if line.startswith('"File Path"'):
            fname = next(csv.reader(io.StringIO(line)))[1].split("/")[-1]
            continue
        if line.startswith('"Line No"'):
            hdr = next(csv.reader(io.StringIO(line)))
            continue
        if hdr is None or line.startswith('"Function Name"'):
            continue
        r = next(csv.reader(io.StringIO(line)))
        if r[0] and r[0] != "":
            d = dict(zip(hdr[2:], r[2:]))
            try:
                inst = int(d.get("Instructions Executed", "0") or 0)
                samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            except ValueError:
                continue
            rows.append((fname, int(r[0]), inst, samp, r[1].strip()[:90]))
    ti = sum(r[2] for r in rows) or 1
    ts = sum(r[3] for r in rows) or 1
    print(f"total warp instructions {ti:,}  stall samples {ts:,}")
    for r in sorted(rows, key=lambda r: -r[3])[:top]:
        print(f"{r[0][:14]:14s}:{r[1]:<5d} inst {100*r[2]/ti:5.1f}%  samp {100*r[3]/ts:5.1f}%  {r[4]}")


if __name__ == "__main__":
    main()
