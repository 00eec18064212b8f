"""Device-resident entry point (the benchmark's timed region).

``ldlt_device`` factors a matrix that already lives in HBM (uint32 residues in
a torch int32 tensor) and leaves P, L, D in HBM: no host copies.  It wraps
``ffb_ldlt_device`` of include/ffldl_b200.h.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from ._lib import lib
from .ffldl import Context, SytrfConfig, _check, _p, default_context


@dataclass
class DeviceFactorization:
    perm: "object"    # torch int32 [n]
    lower: "object"   # torch int32 [n, n] (first `rank` columns valid)
    dkind: "object"   # torch int32 [n]
    dval: "object"    # torch int32 [n]
    dval2: "object"   # torch int32 [n]
    rank: int


class DeviceBuffers:
    """Preallocated outputs, reused across calls."""

    def __init__(self, n: int, device: int = 0):
        import torch
        dev = f"cuda:{device}"
        self.n = n
        self.perm = torch.empty(n, dtype=torch.int32, device=dev)
        self.lower = torch.empty((n, n), dtype=torch.int32, device=dev)
        self.dkind = torch.empty(n, dtype=torch.int32, device=dev)
        self.dval = torch.empty(n, dtype=torch.int32, device=dev)
        self.dval2 = torch.empty(n, dtype=torch.int32, device=dev)


def _after_torch(ctx: Context) -> None:
    """Order the context stream after the work already queued on torch's current stream
    (the input tensors may still be in flight there, e.g. a fresh ``a.clone()``)."""
    import torch
    dev = torch.device("cuda", ctx.device)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(dev))
    torch.cuda.ExternalStream(ctx.stream, device=dev).wait_event(ev)


def ldlt_device(a, field, config: Optional[SytrfConfig] = None, ctx: Optional[Context] = None,
                out: Optional[DeviceBuffers] = None) -> DeviceFactorization:
    """Factor the device matrix ``a`` (n x n int32 tensor of residues; OVERWRITTEN).
    The call runs on the context stream, after the work queued so far on torch's current
    stream, and returns when the factorization is complete."""
    config = config or SytrfConfig()
    p = _p(field)
    ctx = ctx or default_context()
    n = a.shape[0]
    out = out or DeviceBuffers(n, ctx.device)
    _after_torch(ctx)
    rank = C.c_size_t(0)
    _check(lib().ffb_ldlt_device(ctx.handle, p, n, a.data_ptr(), a.stride(0),
                                 int(config.variant), int(config.base_case_threshold),
                                 out.perm.data_ptr(), out.lower.data_ptr(), out.lower.stride(0),
                                 out.dkind.data_ptr(), out.dval.data_ptr(), out.dval2.data_ptr(),
                                 C.byref(rank)))
    return DeviceFactorization(out.perm, out.lower, out.dkind, out.dval, out.dval2, rank.value)


def reconstruction_mismatches(a, fact: DeviceFactorization, field, ctx: Optional[Context] = None) -> int:
    """Entries where P L D L^T P^T != a (blockdiag.hpp:161-182), computed on the device:
    0 proves the factorization reconstructs ``a`` exactly.  ``a`` is the original input
    (n x n int32 residues), left unchanged."""
    p = _p(field)
    ctx = ctx or default_context()
    n = a.shape[0]
    _after_torch(ctx)
    bad = C.c_uint64(0)
    _check(lib().ffb_verify_device(ctx.handle, p, n, a.data_ptr(), a.stride(0), fact.perm.data_ptr(),
                                   fact.lower.data_ptr(), fact.lower.stride(0), fact.dkind.data_ptr(),
                                   fact.dval.data_ptr(), fact.dval2.data_ptr(), fact.rank, C.byref(bad)))
    return int(bad.value)


def pivoting_partners(fact: DeviceFactorization, ctx: Optional[Context] = None):
    """pivoting_matrix (rpmtools.cpp:61-68) as a partner array: int32 tensor, entry i = j
    where Pi(i, j) = 1, else -1."""
    import torch
    ctx = ctx or default_context()
    n = fact.perm.shape[0]
    out = torch.empty(n, dtype=torch.int32, device=fact.perm.device)
    _after_torch(ctx)
    _check(lib().ffb_pivoting_partners_device(ctx.handle, n, fact.perm.data_ptr(), fact.dkind.data_ptr(),
                                              fact.rank, out.data_ptr()))
    return out
