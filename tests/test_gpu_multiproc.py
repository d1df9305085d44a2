"""The replica fan-out across torch.distributed ranks with the real GPU
engine: two processes (gloo for the host-side gather), each running its
np.linspace replica slice on the CUDA engine (engine.py:469-479).  Both
ranks share cuda:0 here -- replica slices never wait on each other, so
this is the multi-rank code path on one device, not a stand-in for a halo
exchange -- and the merged Trajectory must equal the oracle bit for bit,
for the reference xoshiro streams and the bit-plane Philox stream."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


TEMPS = (1.5, 1.9, 2.269, 2.6, 3.0, 3.5, 2.0)


def _worker(rank, world, port, stream, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200.distributed import run_replicas_distributed
    factory = lambda **kw: Engine(device="cuda:0", stream=stream, **kw)  # noqa: E731
    traj = run_replicas_distributed(LatticeDims(32, 1024), TEMPS, 4242, 24, 8, engine_factory=factory)
    out[rank] = (traj.sweeps.tolist(), traj.abs_m.tolist(), traj.energy.tolist(), traj.meta["attempts"],
                 traj.meta["ranks"])
    dist.destroy_process_group()


@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
def test_replica_ranks_on_the_gpu_match_the_oracle(stream):
    from oracle import oracle as orc
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), stream, out), nprocs=world, join=True)
    o = orc.OracleEngine(32, 1024, TEMPS, 4242, stream=stream)
    sw, am, en = o.run(24, 8)
    for r in range(world):
        got_sw, got_m, got_e, att, ranks = out[r]
        assert ranks == world
        assert np.array_equal(np.array(got_sw), sw)
        assert np.array_equal(np.array(got_m), am) and np.array_equal(np.array(got_e), en)
        assert att == o.attempts
