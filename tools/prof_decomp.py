"""torch.profiler table of one decomposed pass at world size 1 (plumbing cost)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1612_06090_b200 import distributed as D, workload  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
w = workload.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
t = [torch.from_numpy(np.ascontiguousarray(w["pos"][:, i].astype(np.float32))).cuda() for i in range(3)]
m = torch.from_numpy(w["mass"]).cuda()
h0 = torch.from_numpy(w["h0"]).cuda()
gid = torch.arange(len(m), device="cuda")
comp = D.LibCompute(0)
for _ in range(2):
    D.decomposed_pass(*t, m, h0, gid, 64, comp, periodic=True, box=w["box"])
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as p:
    D.decomposed_pass(*t, m, h0, gid, 64, comp, periodic=True, box=w["box"])
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(p.key_averages().table(sort_by="cpu_time_total", row_limit=25))
dist.destroy_process_group()
