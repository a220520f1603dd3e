"""Worker of tests/test_sharding.py::test_p2p_exchange_multi_process: G ranks
(processes) row-shard one synthetic DB, share their receive windows by CUDA IPC
and run several sharded searches through the peer-memory exchange; rank 0
checks every epoch against the single-collection search.  Launched with
torch.distributed.run (gloo for the handle all-gather); all ranks may share one
GPU."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_17573_b200 as H  # noqa: E402

N, DIM, B, K, SEED = 7000, 128, 48, 8, 77


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    b0, b1 = H.shard_range(N, world, rank)
    col = H.Collection(DIM, capacity=b1 - b0, device=dev)
    col.generate(H.REAL, SEED, b1 - b0, row0=b0)
    comm = H.Comm(None, world, rank, dev)
    h = comm.p2p_export(B, K)
    handles = [None] * world
    dist.all_gather_object(handles, h)
    comm.p2p_import(handles)
    full = None
    if rank == 0:
        full = H.Collection(DIM, capacity=N, device=dev)
        full.generate(H.REAL, SEED, N)
    ok = True
    for epoch in range(6):
        q = H.gen_queries(H.REAL, 100 + epoch, SEED, N, 0, B - epoch, DIM, device=dev)
        s, i, d = comm.search_topk(col, b0, q, K)
        torch.cuda.synchronize()
        if rank == 0:
            fs, fi = full.search_topk_exact(q, K)
            _, toks = full.keys_view()
            ok &= bool(np.array_equal(i.cpu().numpy(), fi.cpu().numpy()))
            ok &= bool(np.array_equal(s.cpu().numpy(), fs.cpu().numpy()))
            ok &= bool(np.array_equal(d.cpu().numpy(), toks[fi.long()].cpu().numpy()))
        dist.barrier()
    ok &= not comm.p2p_timed_out()
    dist.barrier()
    comm.close()
    if rank == 0:
        print("P2P_OK" if ok else "P2P_MISMATCH", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
