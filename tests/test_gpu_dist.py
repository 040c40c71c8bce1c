"""The W1/L1 re-shard path on the GPU with NCCL (world size 1: this
environment has one GPU per box; the multi-rank host logic is covered on CPU
by test_dist_gloo.py).  Device tensors, the library's CUDA term / mean
kernels and the on-device strong_error partials, against the single-process
reference metrics (oracle) -- bit-identical."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402

from paper_2605_25282_b200 import dist as vdist  # noqa: E402
from paper_2605_25282_b200 import post  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("M,ny,nx", [(11, 3, 7), (64, 20, 50), (1000, 4, 8), (1300, 4, 8)])
def test_nccl_reshard_w1_l1_bit_exact(vo, nccl_group, M, ny, nx):
    rng = np.random.default_rng(M)
    coarse = rng.lognormal(-0.125, 0.5, size=(M, ny, nx))
    fine = rng.lognormal(-0.125, 0.5, size=(M, 2 * ny, 2 * nx))
    # restrict_field (metrics.hpp:29-49): ((f00 + f10) + f01) + f11, times 0.25
    fine_r = (((fine[:, 0::2, 0::2] + fine[:, 0::2, 1::2]) + fine[:, 1::2, 0::2])
              + fine[:, 1::2, 1::2]) * 0.25
    coarse[1, 0, 2] = fine_r[0, 0, 2]  # a tie across ensembles
    coarse, fine_r = coarse.reshape(M, -1), fine_r.reshape(M, -1)
    valid = np.ones(M, bool)
    valid[[0, M - 1]] = False  # jointly invalid samples leave the measure
    dev = torch.device("cuda", 0)
    a = torch.from_numpy(coarse).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(fine_r)).to(dev)
    v = torch.from_numpy(valid).to(dev)
    w1 = vdist.distributed_wasserstein1(torch, dist, a, b, v)
    keep = v.nonzero().reshape(-1)
    ak = a.index_select(0, keep).reshape(-1, ny, nx).contiguous()
    fk = torch.from_numpy(fine[valid]).to(dev).contiguous()
    parts = torch.empty((ak.shape[0], 10), dtype=torch.float64, device=dev)
    post.strong_partials(torch, ak, fk, parts)
    es = vdist.distributed_strong_error(torch, dist, parts)
    n = int(valid.sum())
    A = np.zeros((n, 4, ny, nx))
    B = np.zeros((n, 4, ny, nx))
    A[:, 0] = coarse[valid].reshape(-1, ny, nx)
    B[:, 0] = fine_r[valid].reshape(-1, ny, nx)
    assert float(w1).hex() == vo.wasserstein1(A, B, 0).hex()
    assert float(es).hex() == vo.strong_error(A, B)[0].hex()


def test_bench_sharded_postproc_matches_single_device(nccl_group):
    """bench.py's sharded configs[3] leg (restriction, NCCL re-shard by cell,
    per-cell terms, ordered gather, sequential mean) gives the single-device
    W1 of the same synthetic ensembles, bit for bit."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    M, nxc, nyc = 64, 50, 20
    r = bench.postproc_bench_dist(torch, dist, 0, 1, 0, M=M, nxc=nxc, nyc=nyc, reps=1)
    dev = "cuda:0"
    gen = torch.Generator(device=dev)
    coarse = torch.empty((M, nyc, nxc), dtype=torch.float64, device=dev)
    fine = torch.empty((M, 2 * nyc, 2 * nxc), dtype=torch.float64, device=dev)
    gen.manual_seed(1000)
    coarse.normal_(-0.125, 0.5, generator=gen).exp_()
    gen.manual_seed(1001)
    fine.normal_(-0.125, 0.5, generator=gen).exp_()
    assert float(r["W1"]).hex() == float(post.wasserstein1(torch, coarse, fine)).hex()
    assert r["w1_cells_per_s"] > 0
    assert r["peer"]["identical"] and r["peer"]["w1_cells_per_s"] > 0
