"""Multi-GPU plumbing of the VLBM hot path: one process per
GPU, torch.distributed over NCCL (gloo on CPU for the tests).

* The march shards SAMPLES: rank r owns a contiguous range of sample
  indices (``shard_range``) and marches them with no data-path collective.
* W1 needs every valid sample of a cell together: the density planes of the
  coarse ensemble and of the restricted fine ensemble are re-sharded from
  [samples of rank r] x [all cells] to [all valid samples] x [cells of rank r]
  with ONE all_to_all per ensemble (``reshard_to_cells``).
* The per-cell W1 terms are gathered to rank 0 in rank order, i.e. in cell
  storage order, and summed sequentially there (``ordered_gather``): a tree
  all-reduce would change the summation order and break bit-exactness with
  wasserstein1 (metrics.hpp:112-124).  strong_error's per-sample partials are
  gathered in sample order the same way (metrics.hpp:63-89).

``peer_wasserstein1`` is the fused alternative to the all_to_all: each
rank's W1 kernel reads the other ranks' sample planes directly from their
memory (CUDA IPC peer mappings over NVLink) while it sorts, so the
transfer overlaps the compute and no re-sharded copy is materialised.

Everything here is data movement; the arithmetic runs in the CUDA kernels
(``term_fn`` / ``mean_fn`` arguments default to the device implementations).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block partition: (start, count) of rank's share of n units;
    the first n % world ranks get one extra."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def reshard_to_cells(torch, dist, x_local, counts: Sequence[int], group=None):
    """[m_local, n_cells] (this rank's valid samples, sample-major) ->
    [n_cells_rank, M_total] cell-major columns of ALL valid samples for this
    rank's contiguous cell range, samples in global order (rank order = sample
    order because sample ranges are contiguous).  One all_to_all_single."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m_local, n_cells = x_local.shape
    assert m_local == counts[rank]
    ranges = [shard_range(n_cells, world, q) for q in range(world)]
    # send block for rank q: x_local[:, cells of q], flattened row-major
    send = torch.cat([x_local[:, c0:c0 + cn].reshape(-1) for (c0, cn) in ranges])
    send_splits = [m_local * cn for (_, cn) in ranges]
    my_c0, my_cn = ranges[rank]
    recv_splits = [counts[q] * my_cn for q in range(world)]
    recv = torch.empty(sum(recv_splits), dtype=x_local.dtype, device=x_local.device)
    dist.all_to_all_single(recv, send, recv_splits, send_splits, group=group)
    M = sum(counts)
    return recv.view(M, my_cn).t().contiguous()  # [my_cn, M]


def ordered_gather(torch, dist, x_local, group=None, dst: int = 0):
    """Concatenate 1-D tensors of per-rank lengths on `dst` in rank order
    (returns None on other ranks)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([x_local.numel()], dtype=torch.int64, device=x_local.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    mx = max(ns)
    buf = torch.zeros(mx, dtype=x_local.dtype, device=x_local.device)
    buf[:x_local.numel()] = x_local.reshape(-1)
    out = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, out, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([o[:k] for o, k in zip(out, ns)])


def _device_terms(torch, a_cells, b_cells):
    from . import vlbm as v
    n, M = a_cells.shape
    out = torch.empty(n, dtype=torch.float64, device=a_cells.device)
    if n:
        v._check(v.lib().vlbm_d_w1_cells(M, n, a_cells.data_ptr(), b_cells.data_ptr(),
                                         out.data_ptr(),
                                         torch.cuda.current_stream(a_cells.device).cuda_stream))
    return out


def _device_mean(torch, terms):
    from . import post
    return float(post.ordered_mean(torch, terms).item())


def distributed_wasserstein1(torch, dist, coarse_local, restricted_local, valid_local,
                             term_fn: Optional[Callable] = None,
                             mean_fn: Optional[Callable] = None, group=None):
    """wasserstein1 over the jointly valid samples of a sample-sharded
    ensemble pair.  coarse_local / restricted_local: [m_local, n_cells] planes
    of one variable; valid_local: bool mask [m_local] (joint validity,
    ensemble.hpp:75-91).  Returns W1 on rank 0 (None elsewhere); bit-identical
    to the single-process wasserstein1 over the same valid samples."""
    term_fn = term_fn or (lambda a, b: _device_terms(torch, a, b))
    mean_fn = mean_fn or (lambda t: _device_mean(torch, t))
    world = dist.get_world_size(group)
    keep = valid_local.nonzero().reshape(-1)
    a = coarse_local.index_select(0, keep).contiguous()
    b = restricted_local.index_select(0, keep).contiguous()
    c = torch.tensor([a.shape[0]], dtype=torch.int64, device=a.device)
    cs = [torch.zeros_like(c) for _ in range(world)]
    dist.all_gather(cs, c, group=group)
    counts = [int(v.item()) for v in cs]
    if sum(counts) < 1:
        raise RuntimeError("metrics: no jointly valid samples for pair")
    a_cells = reshard_to_cells(torch, dist, a, counts, group)
    b_cells = reshard_to_cells(torch, dist, b, counts, group)
    terms = term_fn(a_cells, b_cells)
    allterms = ordered_gather(torch, dist, terms, group)
    if allterms is None:
        return None
    return mean_fn(allterms)


_IPC_MAPS: dict = {}  # handle bytes -> [base pointer, open count] (one map per process)


def _ipc_open(L, C, v, hb: bytes) -> int:
    ent = _IPC_MAPS.get(hb)
    if ent is None:
        ptr = C.c_void_p()
        v._check(L.vlbm_ipc_open((C.c_ubyte * 64).from_buffer_copy(hb), C.byref(ptr)))
        ent = _IPC_MAPS[hb] = [ptr.value, 0]
    ent[1] += 1
    return ent[0]


def _ipc_close(L, v, hb: bytes) -> None:
    ent = _IPC_MAPS[hb]
    ent[1] -= 1
    if ent[1] == 0:
        del _IPC_MAPS[hb]
        v._check(L.vlbm_ipc_close(ent[0]))


class PeerRows:
    """Row tables of a sample-sharded ensemble in peer memory: every rank
    exports its planes' allocations with CUDA IPC (vlbm_ipc_handle), the
    handles travel with one all_gather_object, and every rank maps the
    others' allocations (vlbm_ipc_open, peer access over NVLink).  ``rows``
    then lists one device pointer per sample of the whole ensemble in global
    order, wherever the sample lives.  Use as a context manager: leaving it
    barriers (no rank unmaps memory a peer may still read) and unmaps."""

    def __init__(self, torch, dist, planes_local, sample_bytes: int, group=None):
        import ctypes as C

        from . import vlbm as v
        self.torch, self.dist, self.group = torch, dist, group
        self.L, self.C, self.v = v.lib(), C, v
        self.rank = dist.get_rank(group)
        self.opened = []
        h = (C.c_ubyte * 64)()
        off = C.c_uint64()
        m_local = planes_local.shape[0]
        if m_local:
            v._check(self.L.vlbm_ipc_handle(planes_local.data_ptr(), h, C.byref(off)))
        mine = (bytes(h), int(off.value), m_local, torch.cuda.current_device())
        # the planes (often .contiguous() copies made just before, on this
        # rank's stream) must be complete before any peer's kernel reads them:
        # nothing else orders a peer's stream after ours (gloo does not)
        torch.cuda.current_stream().synchronize()
        world = dist.get_world_size(group)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.rows = []
        for q, (hb, offset, mq, dev) in enumerate(allh):
            if mq == 0:
                continue
            if q == self.rank:
                base = planes_local.data_ptr()
            else:
                base = _ipc_open(self.L, C, v, hb) + offset
                self.opened.append(hb)
            self.rows.extend(base + k * sample_bytes for k in range(mq))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.torch.cuda.synchronize()
        self.dist.barrier(group=self.group)  # every peer is done reading
        for hb in self.opened:
            _ipc_close(self.L, self.v, hb)
        self.opened = []


def peer_wasserstein1(torch, dist, coarse_local, fine_local, valid_local, nxc: int,
                      group=None):
    """wasserstein1(coarse, restrict_field(fine)) of one variable over the
    jointly valid samples of a sample-sharded ensemble pair, with NO
    re-shard: each rank computes the terms of its contiguous cell range in
    one kernel that reads every sample's coarse and fine planes where they
    live (vlbm_d_w1_rows over CUDA-IPC peer mappings), so the NVLink
    transfer overlaps the sort; then the per-cell terms go to rank 0 in
    storage order for the sequential mean (bit-identical to the single-
    process wasserstein1).  coarse_local: [m_local, nyc * nxc] float64,
    fine_local: [m_local, 4 * nyc * nxc] (unrestricted), valid_local: bool
    [m_local].  Returns W1 on rank 0, None elsewhere."""
    from . import vlbm as v
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m_local, nc = coarse_local.shape
    if fine_local.shape != (m_local, 4 * nc):
        raise ValueError("wasserstein1: inconsistent field sizes")
    coarse_local, fine_local = coarse_local.contiguous(), fine_local.contiguous()
    vmask = [None] * world
    dist.all_gather_object(vmask, [bool(x) for x in valid_local.tolist()], group=group)
    keep = [k for vm in vmask for k in vm]
    M = sum(keep)
    if M < 1:
        raise RuntimeError("metrics: no jointly valid samples for pair")
    dev = coarse_local.device
    with PeerRows(torch, dist, coarse_local, 8 * nc, group) as cr, \
            PeerRows(torch, dist, fine_local, 32 * nc, group) as fr:
        sel = [i for i, k in enumerate(keep) if k]
        a_rows = torch.tensor([cr.rows[i] for i in sel], dtype=torch.int64, device=dev)
        f_rows = torch.tensor([fr.rows[i] for i in sel], dtype=torch.int64, device=dev)
        c0, cn = shard_range(nc, world, rank)
        terms = torch.empty(cn, dtype=torch.float64, device=dev)
        v._check(v.lib().vlbm_d_w1_rows(M, nxc, c0, cn, a_rows.data_ptr(), f_rows.data_ptr(),
                                        terms.data_ptr(),
                                        torch.cuda.current_stream(dev).cuda_stream))
        if dist.get_backend(group) == "gloo":  # host gather (tests: ranks sharing a GPU)
            terms = terms.cpu()
        allterms = ordered_gather(torch, dist, terms, group)
    if allterms is None:
        return None
    return _device_mean(torch, allterms.to(dev))


def distributed_strong_error(torch, dist, partials_local, group=None,
                             finish_fn: Optional[Callable] = None):
    """strong_error from per-sample partials (M_local x 10, this rank's valid
    samples in order): gathered to rank 0 in sample order and finished there
    exactly as metrics.hpp:81-89."""
    if finish_fn is None:
        from .post import strong_finish
        finish_fn = strong_finish
    allp = ordered_gather(torch, dist, partials_local.reshape(-1), group)
    if allp is None:
        return None
    return finish_fn(allp.view(-1, 10).cpu().numpy())
