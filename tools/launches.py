"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-launch
durations in order (last step only if --tail N) and totals per kernel name."""
import csv, sys, re, collections

path = sys.argv[1]
tail = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"(k_\w+?)(<[^()]*>)?\(", name)
    short = (m.group(1) + (m.group(2) or "")) if m else name[:60]
    rows.append((short, r["Grid Size"], float(r["Metric Value"]) / 1e3))
if tail:
    rows = rows[-tail:]
tot = collections.defaultdict(lambda: [0, 0.0])
for s, g, us in rows:
    print(f"{us:10.1f} us  {g:>16}  {s}")
    tot[s][0] += 1
    tot[s][1] += us
print("---- totals")
for s, (c, us) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{us:10.1f} us  x{c:<4} {s}")
