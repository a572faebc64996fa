"""N > 1 path on CPU: world_size-2 gloo process group, batch-sharded forward (the oracle
network stands in for the device), outputs collected with shard.gather_rows; the result must
be bit-identical to the single-process full-batch forward (A23)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_04071_b200.shard import gather_rows, shard_range

REDUCED = dict(widths=(4, 8, 8, 16), blocks=(1, 1, 1, 1), stem_ch=8, num_classes=10)


def test_shard_range_partitions():
    for total in (0, 1, 5, 256):
        for world in (1, 2, 3, 8):
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import datagen
    from oracle import models
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = datagen.normal(35, 0, (total, 3, 32, 32))
        net = models.ResNetOracle(datagen.lut_randerr(8, 0, 2), 8, config=35, **REDUCED)
        scales = net.calibrate(x[:2])                       # same calibration on every rank
        a, b = shard_range(total, world, rank)
        local = torch.from_numpy(net.forward(x[a:b], scales))
        out = torch.empty(total, REDUCED["num_classes"])
        gather_rows(local, out, total, dist)
        if rank == 0:
            q.put(out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [4, 5])
def test_two_rank_gloo_forward_matches_single_process(total):
    import datagen
    from oracle import models
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x = datagen.normal(35, 0, (total, 3, 32, 32))
    net = models.ResNetOracle(datagen.lut_randerr(8, 0, 2), 8, config=35, **REDUCED)
    ref = net.forward(x, net.calibrate(x[:2]))
    np.testing.assert_array_equal(got, ref)
