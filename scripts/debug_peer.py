"""Debug driver: 2 processes, ShardedChain(transport='peer') on cuda:0."""
import faulthandler
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world, port):
    faulthandler.enable()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1702_02207_b200 import sharded
    rng = np.random.default_rng(21)
    s = 20000
    m, C, x0, v0 = rng.uniform(0.5, 2, s), rng.uniform(500, 2000, s), rng.standard_normal(s), rng.standard_normal(s)
    print(rank, "building", flush=True)
    sh = sharded.ShardedChain(m, C, x0, v0, 1e-3, halo_steps=8, transport="peer")
    print(rank, "built; peers", list(sh.peer_bufs), flush=True)
    for nb, (bufs, nblo) in sh.peer_bufs.items():
        print(rank, "peer", nb, bufs[0][0].device, bufs[0][0].shape, bufs[0][0].data_ptr(), flush=True)
        print(rank, "peer read", float(bufs[0][0][0]), flush=True)
    fb = sh.run(20)
    print(rank, "ran", fb, flush=True)
    sh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(worker, args=(2, port), nprocs=2, join=True, start_method="spawn")
