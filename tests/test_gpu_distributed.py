"""The domain-decomposed pass with the CUDA library as the per-rank compute:
two ranks over gloo sharing the one GPU of this box (host-side collectives
only; no kernel waits on another rank).  Must equal the single-GPU pass."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(n, seed):
    from paper_1612_06090_b200 import workload
    pos, _, _ = workload.nfw_halos(n, 20.0, 10, seed=seed)
    return pos.astype(np.float32), np.random.default_rng(seed).random(n) + 0.5, np.full(n, 0.4)


def _worker(rank, world, port, n, k, out_dir):
    import torch.distributed as dist
    from paper_1612_06090_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, mass, h0 = _data(n, 9)
    sel = np.arange(rank, n, world)
    res = D.density_pass_distributed(pos[sel, 0], pos[sel, 1], pos[sel, 2], mass[sel], h0[sel], sel, k,
                                     D.gpu_local_pass(0), periodic=True, box=20.0)
    np.savez(os.path.join(out_dir, f"g{rank}.npz"), gid=res.gid, h=res.h, rho=res.rho, hist=res.todo_hist)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_match_single_gpu(tmp_path):
    import torch.multiprocessing as mp
    import paper_1612_06090_b200 as sph
    from paper_1612_06090_b200 import distributed as D
    n, k = 30000, 64
    mp.spawn(_worker, args=(2, _port(), n, k, str(tmp_path)), nprocs=2, join=True)
    parts = [np.load(tmp_path / f"g{r}.npz") for r in range(2)]
    gid = np.concatenate([p["gid"] for p in parts])
    assert np.array_equal(np.sort(gid), np.arange(n))
    h = np.empty(n)
    rho = np.empty(n)
    h[gid] = np.concatenate([p["h"] for p in parts])
    rho[gid] = np.concatenate([p["rho"] for p in parts])
    pos, mass, h0 = _data(n, 9)
    want_h, want_rho, _, st = sph.density_pass_soa(pos[:, 0], pos[:, 1], pos[:, 2], mass, h0, k, periodic=True,
                                                   box=20.0)
    assert np.array_equal(h, want_h)
    assert float(np.max(np.abs(rho - want_rho) / want_rho)) <= 1e-4
    assert np.array_equal(D.todo_sizes_from_hist(sum(p["hist"] for p in parts)), st.todo_sizes)
