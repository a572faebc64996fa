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


def _conv_worker(rank, world, port, q):
    """BJ configs[2]-shaped sharding (reduced): rows = images per rank, all_reduce(MAX) of the
    local amax before the scale, all-gather of the outputs.  The oracle stands
    in for the device."""
    import datagen
    import oracle
    from paper_2203_04071_b200.shard import all_reduce_max_
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = datagen.config2(batch=5)
        x = np.ascontiguousarray(c.x[:, :8, :9, :9])
        x[-1] *= np.float32(2.0)             # the global max lives on the last rank's shard
        W = np.ascontiguousarray(c.W[:6, :8])
        a, b = shard_range(x.shape[0], world, rank)
        amax = torch.tensor([float(oracle.amax(x[a:b]))], dtype=torch.float32)
        local_scale = oracle.scale(np.float32(amax.item()), 8)
        all_reduce_max_(amax, dist)
        s = oracle.scale(np.float32(amax.item()), 8)
        qw, sw = oracle.quantize_tensor(W, 8)
        acc = oracle.lut_conv2d(oracle.quantize(x[a:b], s, 8), qw, c.lut, 8, (1, 1), (1, 1))
        local = torch.from_numpy(oracle.dequantize(acc, s, sw, None, 1))
        out = torch.empty((x.shape[0],) + tuple(local.shape[1:]))
        gather_rows(local, out, x.shape[0], dist)
        if rank == 0:
            q.put((out.numpy(), float(s), float(local_scale)))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_conv_amax_allreduce_matches_single_process():
    import datagen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_conv_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, s_used, s_local = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    c = datagen.config2(batch=5)
    x = np.ascontiguousarray(c.x[:, :8, :9, :9])
    x[-1] *= np.float32(2.0)
    W = np.ascontiguousarray(c.W[:6, :8])
    y, _, (_, s_ref, _, _) = oracle.conv2d(x, W, None, c.lut, 8, (1, 1), (1, 1))
    assert s_used == float(s_ref)
    np.testing.assert_array_equal(got, y)
    # the all-reduce matters: rank 0's shard alone has a different amax here
    assert s_local != s_used


def _replica_worker(rank, world, port, q, perturb):
    import datagen
    from paper_2203_04071_b200.shard import verify_replicas
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lut = datagen.lut_randerr(8, 0, 2).copy()
        w = datagen.random_int8(5, (64, 576))
        if perturb and rank == 1:
            lut[12345] += 1
        try:
            verify_replicas([lut, w, np.float32([0.25, 0.5])], dist)
            q.put((rank, "ok"))
        except RuntimeError:
            q.put((rank, "mismatch"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("perturb", [False, True])
def test_replica_checksum_allreduce(perturb):
    """the setup-time checksum all-reduce accepts identical replicas and rejects a
    single differing table entry on one rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q, perturb)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert set(res.values()) == {"mismatch" if perturb else "ok"}
