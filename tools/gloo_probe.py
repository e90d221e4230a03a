"""Probe: which torch.distributed collectives the gloo backend runs on CUDA tensors (dev aid)."""
import os, torch, torch.distributed as dist
dist.init_process_group("gloo")
r = dist.get_rank()
torch.cuda.set_device(0)
out = {}
try:
    t = torch.full((4,), float(r), device="cuda"); dist.all_reduce(t, op=dist.ReduceOp.MAX); out["all_reduce"] = t.tolist()
except Exception as e: out["all_reduce"] = repr(e)[:120]
try:
    s = torch.full((2, 3), r, dtype=torch.uint8, device="cuda"); rv = torch.empty((4, 3), dtype=torch.uint8, device="cuda")
    dist.all_gather_into_tensor(rv, s); out["all_gather_into_tensor"] = rv.tolist()
except Exception as e: out["all_gather_into_tensor"] = repr(e)[:120]
try:
    objs = [None, None]; dist.all_gather_object(objs, r); out["all_gather_object"] = objs
except Exception as e: out["all_gather_object"] = repr(e)[:120]
dist.barrier()
print(r, out, flush=True)
