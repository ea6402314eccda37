"""Probe: can two NCCL ranks share one GPU (for single-GPU tests of the NCCL plane)?"""
import os, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
x = torch.full((4,), rank, device="cuda")
out = torch.empty(4 * world, device="cuda")
dist.all_gather_into_tensor(out, x)
torch.cuda.synchronize()
print(rank, out.tolist(), flush=True)
dist.destroy_process_group()
