"""profiles/ncu_traffic.json from the two k_target full-set captures of a round:
DRAM bytes (read + write) of the seed and main launches, per pass."""
import csv, io, json, subprocess, sys


def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(name)
        tot += float(v[i]) * scale[u[i]]
    return tot


if __name__ == "__main__":
    tag = sys.argv[1]
    cfg_ = sys.argv[2] if len(sys.argv) > 2 else "2"
    seed = dram(f"gpurun_out/{tag}_k_target_c{cfg_}.ncu-rep")
    main = dram(f"gpurun_out/{tag}_k_target_main_c{cfg_}.ncu-rep")
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    json.dump({"config_index": cfg, "k_target_bytes_per_launch": seed + main, "seed_launch_bytes": seed,
               "main_launch_bytes": main,
               "unit": "bytes of DRAM traffic (read + write) of the k_target launches of one pass",
               "source": f"ncu --set full, k_target seed + main launches of config {cfg} ({tag})"},
              open("profiles/ncu_traffic.json", "w"), indent=1)
    print(seed, main)
