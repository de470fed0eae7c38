"""World-size-2/4 CPU (gloo) tests of the SPMD collective host logic.

The product All-Scan moves data in-kernel over peer memory (GPU only); what can
run here is the rank-chain logic shared by the NCCL send/recv baseline and the
LASP-2 all-gather baseline, checked against the oracle's sequential scan
(glasp/collectives.py:70-140 numerics) in both directions.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01004_b200.distributed import AllScanNCCL, lasp2_states

    gen = torch.Generator().manual_seed(11)
    local_all = torch.rand(world, 2, 8, 3, generator=gen, dtype=torch.float64) * 2 - 1
    logs_all = -2 * torch.rand(world, 2, 8, generator=gen, dtype=torch.float64)
    chain = AllScanNCCL()
    out = {}
    for direction in (0, 1):
        r1, s1 = chain(local_all[rank].clone(), logs_all[rank].clone(), 1, direction)
        r2, s2 = lasp2_states(local_all[rank].clone(), logs_all[rank].clone(), direction)
        out[direction] = (r1.numpy(), s1.numpy(), r2.numpy(), s2.numpy())
    results[rank] = (local_all.numpy(), logs_all.numpy(), out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_rank_chain_baselines_match_oracle(world):
    from oracle import gla_oracle as orc

    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    local, logs, _ = results[0]
    for direction in (0, 1):
        order = list(range(world)) if direction == 0 else list(range(world - 1, -1, -1))
        recv, scanned = orc.scan_ranks([local[r] for r in order], [logs[r] for r in order])
        for pos, r in enumerate(order):
            r1, s1, r2, s2 = results[r][2][direction]
            np.testing.assert_allclose(r1, recv[pos], rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(s1, scanned[pos], rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(r2, recv[pos], rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(s2, scanned[pos], rtol=1e-12, atol=1e-14)
