"""NCCL process group with high-priority streams at world size 1 (API check for bench.py's N>1 path)."""
import os
import torch
import torch.distributed as dist
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
opts = dist.ProcessGroupNCCL.Options()
opts.is_high_priority_stream = True
dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
t = torch.ones(4, device="cuda")
dist.all_reduce(t)
s = torch.cuda.Stream(priority=-1)
print("nccl ok", t.tolist(), "stream priority", s.priority, "range", torch.cuda.Stream.priority_range())
dist.destroy_process_group()
