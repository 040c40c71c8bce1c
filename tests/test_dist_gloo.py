"""Multi-rank host logic of the W1/L1 re-shard on CPU (gloo, world_size 2):
sample-sharded ensembles re-sharded by cell with one all_to_all, per-cell W1
terms, ordered gather, sequential mean -- bit-identical to the single-process
reference functions.  (The GPU path swaps in the CUDA term / mean kernels.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_25282_b200 import dist as vdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _terms_cpu(a_cells, b_cells):
    """Per-cell W1 term of metrics.hpp:113-122, sequential in sorted rank."""
    out = torch.empty(a_cells.shape[0], dtype=torch.float64)
    M = a_cells.shape[1]
    for c in range(a_cells.shape[0]):
        sa = sorted(a_cells[c].tolist())
        sb = sorted(b_cells[c].tolist())
        cell = 0.0
        for x, y in zip(sa, sb):
            cell += abs(x - y)
        out[c] = cell / float(M)
    return out


def _mean_cpu(terms):
    acc = 0.0
    for t in terms.tolist():
        acc += t
    return acc / float(terms.numel())


def _partials_cpu(a, b):
    """strong_error per-sample sums (metrics.hpp:69-80), one variable."""
    rows = []
    for m in range(a.shape[0]):
        num = den = 0.0
        for x, y in zip(a[m].tolist(), b[m].tolist()):
            d, r = abs(x - y), abs(y)
            num += d
            den += r
        rows.append([num, den, num, 0.0, 0.0, 0.0, den, 0.0, 0.0, 0.0])
    return torch.tensor(rows, dtype=torch.float64).reshape(-1, 10)


def _worker(rank, world, port, data, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    coarse, fine_r, valid = data
    M = coarse.shape[0]
    s0, cnt = vdist.shard_range(M, world, rank)
    a = torch.from_numpy(coarse[s0:s0 + cnt].copy())
    b = torch.from_numpy(fine_r[s0:s0 + cnt].copy())
    v = torch.from_numpy(valid[s0:s0 + cnt].copy())
    w1 = vdist.distributed_wasserstein1(torch, dist, a, b, v, term_fn=_terms_cpu,
                                        mean_fn=_mean_cpu)
    keep = v.nonzero().reshape(-1)
    parts = _partials_cpu(a.index_select(0, keep), b.index_select(0, keep))
    from paper_2605_25282_b200.post import strong_finish
    es = vdist.distributed_strong_error(torch, dist, parts, finish_fn=strong_finish)
    if rank == 0:
        q.put((w1, es))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_reshard_w1_and_l1_bit_exact(vo, world):
    rng = np.random.default_rng(11)
    M, ny, nx = 11, 3, 7
    coarse = rng.lognormal(-0.125, 0.5, size=(M, ny * nx))
    fine_r = rng.lognormal(-0.125, 0.5, size=(M, ny * nx))
    coarse[3, 5] = fine_r[4, 2]  # a tie across ensembles
    valid = np.ones(M, bool)
    valid[[2, 9]] = False  # jointly invalid samples leave the measure
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), (coarse, fine_r, valid), q),
                       nprocs=world, join=True, start_method="spawn")
    w1, es = q.get(timeout=60)
    # single-process reference over the valid samples (4-component blocks, var 0)
    A = np.zeros((valid.sum(), 4, ny, nx))
    B = np.zeros((valid.sum(), 4, ny, nx))
    A[:, 0] = coarse[valid].reshape(-1, ny, nx)
    B[:, 0] = fine_r[valid].reshape(-1, ny, nx)
    assert float(w1).hex() == vo.wasserstein1(A, B, 0).hex()
    assert float(es).hex() == vo.strong_error(A, B)[0].hex()


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            spans = [vdist.shard_range(n, world, r) for r in range(world)]
            assert sum(c for _, c in spans) == n
            assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(world - 1))
