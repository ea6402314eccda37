"""Debug driver: native p2p all-to-all on thread ranks."""
import sys, traceback, numpy as np, torch
sys.path.insert(0, ".")
from paper_2604_27844_b200 import collectives as coll
from paper_2604_27844_b200.transport import run_ranks
from tests.conftest import rank_words
W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
def body(comm):
    try:
        ok = True
        for it in range(3):
            chunks = [rank_words(comm.rank * 131 + q, 2000, seed=it) for q in range(W)]
            spec = coll.AlltoAllSpec(chunks, [2000] * W)
            z = coll.zip_all_to_all_d2(comm, spec)
            print(comm.rank, it, "zip done", flush=True)
            r = coll.reference_all_to_all(comm, spec)
            ok &= all(torch.equal(a, b) for a, b in zip(z, r))
        return ok
    except Exception:
        print(comm.rank, traceback.format_exc(), flush=True)
        raise
print(run_ranks(W, body), flush=True)
