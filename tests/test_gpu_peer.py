"""W1 with the samples left where they live (dist.peer_wasserstein1): each
rank's kernel reads the other ranks' sample planes through CUDA IPC peer
mappings instead of an all_to_all re-shard (vlbm_d_w1_rows, restriction
fused).  One GPU per box here, so the multi-rank case runs two processes on
the same device -- real IPC mappings between processes, no kernel waits on
another rank -- with a gloo group for the host exchange; the result must be
the single-process wasserstein1(coarse, restrict_field(fine)) bit for bit."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ensemble(M, nyc, nxc, seed):
    rng = np.random.default_rng(seed)
    c = rng.lognormal(-0.125, 0.5, size=(M, nyc * nxc))
    f = rng.lognormal(-0.125, 0.5, size=(M, 4 * nyc * nxc))
    valid = np.ones(M, bool)
    valid[[1, M - 2]] = False  # jointly invalid samples leave the measure
    return c, f, valid


def _single(M, nyc, nxc, seed):
    from paper_2605_25282_b200 import post
    c, f, valid = _ensemble(M, nyc, nxc, seed)
    tc = torch.from_numpy(c[valid].reshape(-1, nyc, nxc)).cuda()
    tf = torch.from_numpy(f[valid].reshape(-1, 2 * nyc, 2 * nxc)).cuda()
    return float(post.wasserstein1(torch, tc, tf))


def _worker(rank, world, port, M, nyc, nxc, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_25282_b200 import dist as vd
    c, f, valid = _ensemble(M, nyc, nxc, seed)
    s0, m = vd.shard_range(M, world, rank)
    tc = torch.from_numpy(c[s0:s0 + m]).cuda()
    tf = torch.from_numpy(f[s0:s0 + m]).cuda()
    tv = torch.from_numpy(valid[s0:s0 + m])
    w1 = vd.peer_wasserstein1(torch, dist, tc, tf, tv, nxc)
    if rank == 0:
        out.put(float(w1).hex())
    dist.destroy_process_group()


@pytest.mark.parametrize("M,nyc,nxc", [(37, 6, 10), (1100, 4, 6)])
def test_peer_w1_one_rank(M, nyc, nxc):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        from paper_2605_25282_b200 import dist as vd
        c, f, valid = _ensemble(M, nyc, nxc, 5)
        w1 = vd.peer_wasserstein1(torch, dist, torch.from_numpy(c).cuda(),
                                  torch.from_numpy(f).cuda(), torch.from_numpy(valid), nxc)
    finally:
        dist.destroy_process_group()
    assert float(w1).hex() == float(_single(M, nyc, nxc, 5)).hex()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_w1_ranks_share_gpu(world):
    M, nyc, nxc, seed = 45, 6, 10, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, nyc, nxc, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == float(_single(M, nyc, nxc, seed)).hex()
