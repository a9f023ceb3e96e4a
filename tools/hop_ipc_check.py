"""Two PROCESSES, one GPU: the device-initiated coarse-chain hop over cudaIpc mappings
(HopComm.over_ipc) against the single-engine run, bit for bit.  The ranks' kernels never
wait on one another (the receiver's *stream* waits on the flag), so sharing one GPU is safe.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29611 tools/hop_ipc_check.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2304_14074_b200 import _native as N  # noqa: E402
from paper_2304_14074_b200 import distributed as D  # noqa: E402
from paper_2304_14074_b200 import grid as G  # noqa: E402
from paper_2304_14074_b200 import parareal as P  # noqa: E402
from paper_2304_14074_b200.configs import CONFIGS, initial_condition  # noqa: E402
from paper_2304_14074_b200.engine import PararealEngine  # noqa: E402


class CpuRed:
    """increment all-reduce through host tensors (gloo)"""
    def __init__(self, world): self.world = world
    def all_reduce_max(self, t, async_op=False):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        t.copy_(h)
        return None


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    out = {}
    for cfg, nsl, J, max_iter in ((3, 8, 32, 4), (2, 8, 512, 6)):
        c = CONFIGS[cfg]
        g = G.SpatialGrid(c["dim"], c["nx"])
        dT = c["T"] / c["N"]
        part = P.TimePartition(nsl * dT, nsl, J)
        var = P.AlgorithmVariant(c["variant"])
        f, co = P.propagator_pair(var, part, c["eps"])
        u0 = initial_condition(cfg)
        ctx = N.Context.get(0)
        comm = D.HopComm.over_ipc(ctx, rank, world, 1, g.device_size)
        comm.red = CpuRed(world)
        sh = D.ShardedParareal(g, f, co, nsl, J, rank=rank, world=world, comm=comm)
        sh.load(G.Field(g, u0))
        sh.run(max_iter=max_iter, pipelined=False)
        torch.cuda.synchronize()
        loc = sh.local_iterates(0)
        parts = [None] * world
        dist.all_gather_object(parts, loc)
        if rank == 0:
            eng = PararealEngine(g, f, co, nsl, J)
            eng.load([G.Field(g, u0)])
            eng.run(max_iter=max_iter)
            ref = eng.iterates_host(0)
            got = np.concatenate(parts)
            out[f"config{cfg}_trunc"] = {"bit_identical": bool(np.array_equal(ref, got)),
                                         "k": sh.k, "increments_equal": bool(
                                             np.array_equal(np.array(sh.increments), np.array([x[0] for x in eng.increments])))}
        dist.barrier()
    if rank == 0:
        print(json.dumps({"hop_over_ipc_two_processes_one_gpu": out}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
