"""Randomised check of the domain decomposition on one GPU (run on a GPU box):
random sets, random world sizes (in-process ranks, ThreadComm, private
library contexts), random initial splits; the decomposed h must equal the
one-GPU pass bit for bit and the todo traces must add up.

    python tools/fuzz_decomp.py [cases] [seed]
"""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1612_06090_b200 import distributed as D  # noqa: E402
from paper_1612_06090_b200 import workload  # noqa: E402
from paper_1612_06090_b200.density import density_pass_soa  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
    bad = 0
    for c in range(cases):
        world = int(rng.choice([2, 3, 4, 5, 8]))
        n = int(rng.integers(2000, 60000))
        k = int(rng.choice([16, 32, 64, 128]))
        box = float(rng.choice([10.0, 100.0]))
        periodic = bool(rng.random() < 0.6)
        kind = rng.choice(["nfw", "uniform", "blobs"])
        if kind == "nfw":
            pos, _, _ = workload.nfw_halos(n, box, int(rng.integers(1, 40)), seed=int(rng.integers(1 << 30)))
        elif kind == "uniform":
            pos = (rng.random((n, 3)) * box).astype(np.float32).astype(np.float64)
        else:
            cc = rng.random((4, 3)) * box
            pos = np.mod(cc[rng.integers(0, 4, n)] + rng.normal(0, box * 0.02, (n, 3)), box)
            pos = pos.astype(np.float32).astype(np.float64)
            pos[pos >= box] = np.float64(np.nextafter(np.float32(box), np.float32(0.0)))
        p32 = pos.astype(np.float32)
        mass = rng.random(n) + 0.5
        h0 = np.full(n, workload._initial_h(box, n, k))
        h_ref, rho_ref, _, st = density_pass_soa(p32[:, 0], p32[:, 1], p32[:, 2], mass, h0, k, periodic=periodic,
                                                 box=box)
        split = rng.permutation(n) if rng.random() < 0.5 else np.arange(n)
        parts = np.array_split(split, world)
        W = D.ThreadWorld(world)
        out, errs = [None] * world, []

        def run(r):
            try:
                sel = np.sort(parts[r])
                comp = D.LibCompute(0, private_context=True)
                t = [torch.from_numpy(np.ascontiguousarray(p32[sel, i])).cuda() for i in range(3)]
                out[r] = D.decomposed_pass(*t, torch.from_numpy(mass[sel]).cuda(), torch.from_numpy(h0[sel]).cuda(),
                                           torch.from_numpy(sel.astype(np.int64)).cuda(), k, comp,
                                           periodic=periodic, box=box, comm=D.ThreadComm(W, r))
                torch.cuda.synchronize()
            except Exception as e:
                errs.append(repr(e))
                W.barrier.abort()

        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        [t.start() for t in th]
        [t.join() for t in th]
        if errs:
            print(c, "BAD", errs[:1], flush=True)
            bad += 1
            continue
        gid = np.concatenate([o.gid.cpu().numpy() for o in out])
        h = np.empty(n)
        rho = np.empty(n)
        h[gid] = np.concatenate([o.h.cpu().numpy() for o in out])
        rho[gid] = np.concatenate([o.rho.cpu().numpy() for o in out])
        todo = D.todo_sizes_from_hist(sum(o.todo_hist for o in out))
        ok = (np.array_equal(np.sort(gid), np.arange(n)) and np.array_equal(h, h_ref)
              and float(np.max(np.abs(rho - rho_ref) / rho_ref)) < 1e-5 and np.array_equal(todo, st.todo_sizes))
        bad += not ok
        print(f"{c:3d} {'ok ' if ok else 'BAD'} {kind:7s} world={world} n={n:6d} k={k:3d} periodic={periodic!s:5s} "
              f"ghosts={sum(o.n_ghosts for o in out) / n:.2f}x h_mis={int(np.sum(h != h_ref))}", flush=True)
    print(f"{cases - bad}/{cases} ok")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
