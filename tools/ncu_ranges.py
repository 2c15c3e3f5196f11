"""Aggregate an ncu source page by line ranges of one file:
python tools/ncu_ranges.py REP FILE name:a-b name:a-b ..."""
import subprocess, csv, io, sys
rep, fn = sys.argv[1], sys.argv[2]
ranges = {}
for spec in sys.argv[3:]:
    k, ab = spec.split(":"); a, b = ab.split("-"); ranges[k] = (int(a), int(b))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []; fname = "?"; hdr = None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        fname = next(csv.reader(io.StringIO(line)))[1].split("/")[-1]; continue
    if line.startswith('"Line No"'):
        hdr = next(csv.reader(io.StringIO(line))); continue
    if hdr is None or line.startswith('"Function Name"'): continue
    r = next(csv.reader(io.StringIO(line)))
    if r[0]:
        d = dict(zip(hdr[2:], r[2:]))
        try:
            inst = int(d.get("Instructions Executed", "0") or 0); samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        rows.append((fname, int(r[0]), inst, samp))
ti = sum(r[2] for r in rows) or 1; ts = sum(r[3] for r in rows) or 1
agg = {k: [0, 0] for k in ranges}; other = [0, 0]
for f, l, i, s in rows:
    for k, (a, b) in ranges.items():
        if f == fn and a <= l <= b:
            agg[k][0] += i; agg[k][1] += s; break
    else:
        other[0] += i; other[1] += s
print(f"total inst {ti:,}  samples {ts:,}")
for k, (i, s) in agg.items():
    print(f"{k:10s} inst {100*i/ti:5.1f}%  samp {100*s/ts:5.1f}%")
print(f"{'other':10s} inst {100*other[0]/ti:5.1f}%  samp {100*other[1]/ts:5.1f}%")
