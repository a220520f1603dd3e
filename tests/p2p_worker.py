"""Worker of tests/test_sharding.py's multi-process exchange tests: G ranks
(processes) row-shard one synthetic DB and run several sharded searches
(hsd_search_topk_sharded) through
  --exchange p2p:  the peer-memory exchange (receive windows shared by CUDA IPC;
                   all ranks may share one GPU), or
  --exchange nccl: the product's NCCL all-gather communicator (hsd_comm_create;
                   one GPU per rank when the box has them — NCCL refuses two
                   ranks on one device, reported as NCCL_SAME_DEVICE);
rank 0 checks every epoch against the single-collection search.  Launched with
torch.distributed.run (gloo carries the handles / the NCCL unique id)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_17573_b200 as H  # noqa: E402

N, DIM, B, K, SEED = 7000, 128, 48, 8, 77


def main():
    exchange = sys.argv[sys.argv.index("--exchange") + 1] if "--exchange" in sys.argv else "p2p"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    b0, b1 = H.shard_range(N, world, rank)
    col = H.Collection(DIM, capacity=b1 - b0, device=dev)
    col.generate(H.REAL, SEED, b1 - b0, row0=b0)
    if exchange == "nccl":
        uid = [H.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        devs = [None] * world
        dist.all_gather_object(devs, str(torch.cuda.get_device_properties(dev).uuid))
        if len(set(devs)) < world:
            if rank == 0:
                print("NCCL_SAME_DEVICE", flush=True)
            dist.destroy_process_group()
            return
        comm = H.Comm(uid[0], world, rank, dev)
        print(f"rank {rank}: data-path NCCL communicator with {comm.world} ranks", flush=True)
    else:
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
    if exchange == "p2p":
        ok &= not comm.p2p_timed_out()
    dist.barrier()
    comm.close()
    if rank == 0:
        tag = "P2P" if exchange == "p2p" else "NCCL"
        print(f"{tag}_OK" if ok else f"{tag}_MISMATCH", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
