"""Probe: does torch.distributed gloo exchange CUDA tensors with batch_isend_irecv / all_gather?"""
import os
import torch
import torch.distributed as dist
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
x = torch.full((4, 3), float(r), device="cuda")
y = torch.empty_like(x)
reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, x, (r + 1) % w), dist.P2POp(dist.irecv, y, (r - 1) % w)])
for q in reqs:
    q.wait()
outs = [torch.empty_like(x) for _ in range(w)]
dist.all_gather(outs, x)
print(r, y[0, 0].item(), [o[0, 0].item() for o in outs], flush=True)
dist.destroy_process_group()
