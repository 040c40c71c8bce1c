"""Device-resident W1/L1 post-processing on torch CUDA tensors (torch is only
the allocator/stream plumbing; every number comes from post.cu via the C ABI).

The ensemble layout is sample-major planes of one variable: ``coarse`` is
(M, nyc, nxc), ``fine`` is (M, 2*nyc, 2*nxc), both float64 on one device.
The restriction of the fine ensemble (restrict_field, metrics.hpp:29-49) is
fused into both reductions.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .vlbm import _check, lib


def _ptr(t) -> int:
    return t.data_ptr()


def _stream(torch, t) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _check_pair(coarse, fine):
    if coarse.dtype != fine.dtype or str(coarse.dtype) != "torch.float64":
        raise ValueError("expected float64 tensors")
    M, nyc, nxc = coarse.shape
    if fine.shape != (M, 2 * nyc, 2 * nxc):
        raise ValueError("wasserstein1: inconsistent field sizes")
    if not (coarse.is_contiguous() and fine.is_contiguous()):
        raise ValueError("expected contiguous tensors")
    return M, nyc, nxc


def w1_cell_terms(torch, coarse, fine, out=None):
    """Per-cell W1 terms sum_m |a_(m) - b_(m)| / M (metrics.hpp:113-122)."""
    M, nyc, nxc = _check_pair(coarse, fine)
    if out is None:
        out = torch.empty(nyc * nxc, dtype=torch.float64, device=coarse.device)
    _check(lib().vlbm_d_w1_restrict(M, nxc, nyc, _ptr(coarse), nyc * nxc, _ptr(fine),
                                    4 * nyc * nxc, _ptr(out), _stream(torch, coarse)))
    return out


def ordered_mean(torch, terms, out=None):
    """Storage-order sequential mean of the per-cell terms (bit-exact acc)."""
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=terms.device)
    _check(lib().vlbm_d_ordered_mean(terms.numel(), _ptr(terms), _ptr(out),
                                     _stream(torch, terms)))
    return out


def w1_mean(torch, coarse, fine, out=None, terms=None):
    """wasserstein1(coarse, restrict(fine)) on the device: per-cell terms and
    the storage-order mean in one call, the sequential mean overlapped with
    the terms chunk by chunk (bit-identical to w1_cell_terms + ordered_mean)."""
    M, nyc, nxc = _check_pair(coarse, fine)
    if terms is None:
        terms = torch.empty(nyc * nxc, dtype=torch.float64, device=coarse.device)
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=coarse.device)
    _check(lib().vlbm_d_w1_restrict_mean(M, nxc, nyc, _ptr(coarse), nyc * nxc, _ptr(fine),
                                         4 * nyc * nxc, _ptr(terms), _ptr(out[1:]), _ptr(out),
                                         _stream(torch, coarse)))
    return out[:1]


def wasserstein1(torch, coarse, fine) -> float:
    """wasserstein1(coarse, restrict(fine)) over one variable (bit-exact)."""
    return float(w1_mean(torch, coarse, fine).item())


def strong_partials(torch, coarse, fine, out=None):
    """Per-sample (num, den, cnum[4], cden[4]) of strong_error in the
    reference's sequential order, one variable, restriction fused."""
    M, nyc, nxc = _check_pair(coarse, fine)
    if out is None:
        out = torch.empty((M, 10), dtype=torch.float64, device=coarse.device)
    _check(lib().vlbm_d_strong_partials_var(M, nxc, nyc, _ptr(coarse), nyc * nxc, _ptr(fine),
                                            4 * nyc * nxc, _ptr(out), _stream(torch, coarse)))
    return out


def strong_finish(partials) -> float:
    p = np.ascontiguousarray(partials, np.float64)
    r = C.c_double()
    pc = np.zeros(4)
    _check(lib().vlbm_strong_finish(p.shape[0], p.ctypes.data_as(C.POINTER(C.c_double)),
                                    C.byref(r), pc.ctypes.data_as(C.POINTER(C.c_double))))
    return r.value


def strong_error(torch, coarse, fine) -> float:
    """strong_error(coarse, restrict(fine)) when only this variable is nonzero."""
    return strong_finish(strong_partials(torch, coarse, fine).cpu().numpy())


def pair_metrics(coarse, fine, var: int = 0, batch: int = 0, device: int = 0):
    """compute_metrics' (W1, E_strong) of one grid pair and time through the
    C ABI's vlbm_metrics_* (one upload per ensemble, restriction fused, all
    reductions on the device): host fields coarse (M, 4, nyc, nxc), fine
    (M, 4, 2 nyc, 2 nxc), added in batches of ``batch`` samples (0: all)."""
    c = np.ascontiguousarray(coarse, np.float64)
    f = np.ascontiguousarray(fine, np.float64)
    M, _, nyc, nxc = c.shape
    if f.shape != (M, 4, 2 * nyc, 2 * nxc):
        raise ValueError("wasserstein1: inconsistent field sizes")
    L = lib()
    h = C.c_void_p()
    _check(L.vlbm_metrics_begin(M, nxc, nyc, int(var), device, C.byref(h)))
    try:
        b = batch or M
        dp = C.POINTER(C.c_double)
        for s0 in range(0, M, b):
            nb = min(b, M - s0)
            _check(L.vlbm_metrics_add(h, s0, nb, c[s0:s0 + nb].ctypes.data_as(dp),
                                      f[s0:s0 + nb].ctypes.data_as(dp)))
        w1, es = C.c_double(), C.c_double()
        _check(L.vlbm_metrics_finish(h, C.byref(w1), C.byref(es), None))
        return w1.value, es.value
    finally:
        L.vlbm_metrics_destroy(h)
