"""Two ranks of the device path on ONE GPU (cuda:0): each process runs the batch-sharded
ApproxResNet forward on its shard with its own kernels, the ranks verify their replicated state
(checksum all-reduce) and collect the logits with shard.gather_rows over gloo (host-staged
copies).  The kernels of the two ranks never wait on each other -- only the host-side
collectives synchronise them -- so this is a faithful functional test of the N > 1 product path
 that one GPU can run.  The gathered logits must be bit-identical to the
single-process full-batch forward and to the oracle (A23)."""
import os
import socket

import numpy as np
import pytest
import torch

import datagen
from oracle import models

pytestmark = pytest.mark.gpu
REDUCED = dict(widths=(16, 32, 16, 32), blocks=(1, 2, 1, 1), stem_ch=16, num_classes=24)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _images(full, total):
    return datagen.config3_images(total) if full else datagen.normal(37, 0, (total, 3, 40, 36))


def _net(full, lut_np):
    from paper_2203_04071_b200 import Lut
    from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs
    topo = {} if full else REDUCED
    W = datagen.network_weights(layer_specs(**topo), 3 if full else 37)
    return ApproxResNet(W, Lut(8, lut_np), "cuda", **topo)


def _worker(rank, world, port, total, full, q):
    import torch.distributed as dist
    from paper_2203_04071_b200 import _lib
    from paper_2203_04071_b200.shard import gather_rows, shard_range, verify_replicas
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lut = datagen.lut_randerr(8, 0, 2)
        net = _net(full, lut)
        x = torch.from_numpy(_images(full, total)).cuda()
        net.calibrate(x[:2])                                 # identical static scales per rank
        verify_replicas(net.replicated_state() + [torch.from_numpy(lut)], dist, device="cuda")
        a, b = shard_range(total, world, rank)
        lg = net.forward(x[a:b])
        kern = _lib.axq_last_path()[0]
        out = torch.empty(total, lg.shape[1], device="cuda")
        gather_rows(lg, out, total, dist)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy(), kern))
    except Exception as e:      # surface the failure in the parent
        q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("full,total", [(False, 5), (True, 8)], ids=["reduced-uneven", "c3-shapes"])
def test_two_ranks_one_gpu_sharded_resnet(full, total):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, full, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, out, kern = q.get(timeout=600)
        res[r] = (out, kern)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, res
    assert isinstance(res[0][0], np.ndarray), res[0][0]
    np.testing.assert_array_equal(res[0][0], res[1][0])          # every rank holds all rows
    lut = datagen.lut_randerr(8, 0, 2)
    net = _net(full, lut)
    x = _images(full, total)
    xd = torch.from_numpy(x).cuda()
    net.calibrate(xd[:2])
    single = net.forward(xd).cpu().numpy()
    np.testing.assert_array_equal(res[0][0], single)               # G = 2 == G = 1
    orc = models.ResNetOracle(lut, 8, config=3 if full else 37, **({} if full else REDUCED))
    scales = orc.calibrate(x[:2])
    for i in ((0, total - 1) if full else range(total)):
        np.testing.assert_array_equal(res[0][0][i:i + 1], orc.forward(x[i:i + 1], scales))
