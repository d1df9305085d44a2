"""Probe: can two processes on ONE GPU rendezvous torch symmetric memory over
a gloo group and read each other's buffers (no kernel waits on another)?"""
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch.distributed._symmetric_memory as symm_mem
    try:
        buf = symm_mem.empty(1024, dtype=torch.int32, device="cuda:0")
        buf.fill_(100 + rank)
        torch.cuda.synchronize()
        h = symm_mem.rendezvous(buf, dist.group.WORLD)
        dist.barrier()
        peer = (rank + 1) % world
        ptr = int(h.buffer_ptrs[peer])
        # read the peer's buffer through its mapping with a device copy
        import ctypes
        cudart = ctypes.CDLL("libcudart.so")
        out = torch.empty(1024, dtype=torch.int32, device="cuda:0")
        rc = cudart.cudaMemcpy(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ptr), ctypes.c_size_t(4096), 3)
        torch.cuda.synchronize()
        print(f"rank {rank}: rendezvous ok, peer ptr {ptr:#x}, memcpy rc {rc}, peer value {int(out[0])}", flush=True)
    except Exception as exc:
        print(f"rank {rank}: {type(exc).__name__}: {exc}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(2, port), nprocs=2, join=True)
