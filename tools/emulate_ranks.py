"""The decomposed multi-GPU pass with WORLD in-process ranks on one GPU
(threads, ThreadComm, one private library context per rank).

Checks the result against the single-GPU pass over the whole set (h bit for
bit, density to the fp32 sum order) and reports the decomposition's shape
(owned / ghost counts per rank) plus each rank's final pass re-timed ALONE on
the GPU (CUDA events), i.e. the per-rank compute a WORLD-GPU run would see.

    python tools/emulate_ranks.py CONFIG WORLD [--json out.json]
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1612_06090_b200 import distributed as D, workload  # noqa: E402
from paper_1612_06090_b200.density import density_pass_soa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("world", type=int)
    ap.add_argument("--json", default=None)
    ap.add_argument("--group", type=int, default=256)
    args = ap.parse_args()
    world = args.world
    t0 = time.time()
    w = workload.config_weak(args.config, world)
    n, k, box = w["pos"].shape[0], int(w["k"]), float(w["box"])
    pos32 = w["pos"].astype(np.float32)
    print(f"config {args.config} x{world}: n={n} box={box:.2f} (gen {time.time() - t0:.1f}s)", flush=True)

    # single-GPU reference over the whole set
    h_ref, rho_ref, _, st = density_pass_soa(pos32[:, 0], pos32[:, 1], pos32[:, 2], w["mass"], w["h0"], k,
                                             periodic=True, box=box)
    t_single = st.device["t_stage_ms"]["total"]
    # the whole-set context is large (C4: ~40 GB): free it before the ranks build theirs
    from paper_1612_06090_b200 import _lib
    _lib.drop_context(0)
    torch.cuda.empty_cache()

    W = D.ThreadWorld(world)
    out, comps, errs = [None] * world, [None] * world, []

    def run(r):
        try:
            sel = np.arange(r, n, world)
            c = D.LibCompute(0, private_context=True)
            c.keep_inputs = True
            comps[r] = c
            t = [torch.from_numpy(np.ascontiguousarray(pos32[sel, i])).cuda() for i in range(3)]
            res = D.decomposed_pass(*t, torch.from_numpy(w["mass"][sel]).cuda(), torch.from_numpy(w["h0"][sel]).cuda(),
                                    torch.from_numpy(sel.astype(np.int64)).cuda(), k, c, periodic=True, box=box,
                                    comm=D.ThreadComm(W, r), group_particles=args.group)
            torch.cuda.synchronize()
            out[r] = res
        except Exception as e:
            errs.append(repr(e))
            W.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    t1 = time.time()
    [t.start() for t in th]
    [t.join() for t in th]
    if errs:
        raise SystemExit(f"rank failure: {errs}")
    print(f"decomposed pass done ({time.time() - t1:.1f}s wall, ranks concurrent on one GPU)", flush=True)
    gid = np.concatenate([o.gid.cpu().numpy() for o in out])
    assert np.array_equal(np.sort(gid), np.arange(n)), "ownership is not a partition"
    h = np.empty(n)
    rho = np.empty(n)
    h[gid] = np.concatenate([o.h.cpu().numpy() for o in out])
    rho[gid] = np.concatenate([o.rho.cpu().numpy() for o in out])
    h_mis = int(np.sum(h != h_ref))
    rho_rel = float(np.max(np.abs(rho - rho_ref) / rho_ref))

    # each rank's final pass alone
    per_rank = []
    for r in range(world):
        c = comps[r]
        inp = c.last_inputs
        ms = []
        for rep in range(3):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(c.stream):
                s.record()
                c.local_pass(*inp)
                e.record()
            e.synchronize()
            ms.append(s.elapsed_time(e))
        tk = c.last_stats["t_kernel_ms"]
        per_rank.append({"owned": out[r].n_owned, "ghosts": out[r].n_ghosts, "max_bound": out[r].max_bound,
                         "final_pass_ms": min(ms), "tree_ms": tk["tree"], "search_ms": tk["search"],
                         "pair_tests": c.last_stats["pair_tests"]})
    # how tight are the bounds?  bound / h over all owned particles
    ratio = np.concatenate([(o.bound / o.h).cpu().numpy() for o in out])
    qs = np.quantile(ratio, [0.5, 0.9, 0.99, 0.999, 1.0]).tolist()
    # rank 0's ghost marking alone
    c = comps[0]
    gm = []
    for rep in range(3):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(c.stream):
            s.record()
            c.ghost_mask(*c.last_ghost_inputs)
            e.record()
        e.synchronize()
        gm.append(s.elapsed_time(e))
    res = {"config": args.config, "ghost_mask_ms_rank0": min(gm), "bound_over_h_quantiles_50_90_99_999_max": qs,
           "n_groups_rank0": int(c.last_ghost_inputs[0].shape[0]), "n_foreign_rank0": int(c.last_ghost_inputs[4].shape[0]), "world": world, "n": n, "h_mismatches": h_mis, "rho_max_rel": rho_rel,
           "single_gpu_pass_ms": t_single, "per_rank": per_rank,
           "final_pass_ms_max": max(p["final_pass_ms"] for p in per_rank),
           "ghost_fraction": sum(p["ghosts"] for p in per_rank) / n}
    print(json.dumps(res, indent=1))
    if args.json:
        json.dump(res, open(args.json, "w"), indent=1)
    return 0 if h_mis == 0 and rho_rel < 1e-5 else 1


if __name__ == "__main__":
    sys.exit(main())
