"""Debug driver: native local group, one all-gather per plane."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2604_27844_b200.native import NativeComm
from paper_2604_27844_b200 import collectives as coll
from paper_2604_27844_b200.transport import run_ranks
print("creating", flush=True)
cs = NativeComm.local_group(2)
print("created", [ (c.rank, c.world_size, c.p2p_available, c.shared_device) for c in cs], flush=True)
for c in cs: c.close()
print("closed", flush=True)
def body(comm):
    x = torch.randn(100000, device="cuda").to(torch.bfloat16)
    print("rank", comm.rank, "ag", flush=True)
    z = coll.zip_all_gather(comm, x)
    r = coll.reference_all_gather(comm, x)
    return bool(torch.equal(z, r))
print(run_ranks(2, body), flush=True)
