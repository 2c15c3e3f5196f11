"""profiles/ncu_traffic.json from the full-set captures of a round's search
launches (tools/gpu_ncu_c3.sh): DRAM bytes (read + write) of the k_target launch
over the calibration sample, the k_lane launch and the k_target launch over
what k_lane leaves, per pass, plus their issue-slot utilisation."""
import csv, io, json, subprocess, sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def dram(rep):
    h, u, v = raw(rep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(name)
        tot += float(v[i]) * scale[u[i]]
    return tot


def metric(rep, name):
    h, u, v = raw(rep)
    return float(v[h.index(name)]) if name in h else None


def duration_ms(rep):
    h, u, v = raw(rep)
    i = h.index("gpu__time_duration.sum")
    return float(v[i]) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(u[i], 1.0)


if __name__ == "__main__":
    tag = sys.argv[1]
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    reps = {k: f"gpurun_out/{tag}_{k}_c{cfg}.ncu-rep" for k in ("k_target_sample", "k_lane", "k_target_rest")}
    b = {k: dram(r) for k, r in reps.items()}
    busy = {k: metric(r, "sm__inst_issued.avg.pct_of_peak_sustained_active") for k, r in reps.items()}
    inst = {k: metric(r, "smsp__inst_executed.sum") for k, r in reps.items()}
    ms = {k: duration_ms(r) for k, r in reps.items()}
    json.dump({"config_index": cfg, "search_bytes_per_launch": sum(b.values()), "launch_bytes": b,
               "unit": "bytes of DRAM traffic (read + write) of the search launches of one pass "
                       "(k_target calibration sample + k_lane + k_target leftovers)",
               "source": f"ncu --set full of config {cfg} ({tag}), one capture per launch",
               "issue_slots_busy": {k: (v / 100.0 if v is not None else None) for k, v in busy.items()},
               "warp_instructions": inst, "ncu_ms": ms},
              open("profiles/ncu_traffic.json", "w"), indent=1)
    print(b, busy, inst, ms)
