"""The five benchmark configurations of BASELINE.json and their generators.

Inputs are seeded counter-based functions of (seed, i, j) (csrc/ffb_gen.cu),
so the host generator (uint64, for the CPU oracle) and the device generator
(uint32 in HBM, for the engine) produce identical matrices at any size.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._lib import lib
from .ffldl import _check


@dataclass(frozen=True)
class Workload:
    config: int
    n: int
    p: int
    r: int  # rank parameter (configs 2 and 5), else 0
    seed: int
    description: str

    def scaled(self, n: int) -> "Workload":
        """Same family at another size (rank parameter scaled with n)."""
        r = (self.r * n) // self.n if self.r else 0
        return Workload(self.config, n, self.p, r, self.seed, self.description)


CONFIGS = {
    1: Workload(1, 1024, 131, 0, 1, "dense symmetric, uniform [0,130]"),
    2: Workload(2, 4096, 131, 2048, 2, "M diag(d) M^T, rank 2048, symmetric row permutation"),
    3: Workload(3, 8192, 8388593, 0, 3, "dense symmetric, uniform [0,p-1], p = 8388593"),
    4: Workload(4, 16384, 131, 0, 4, "hollow symmetric (zero diagonal)"),
    5: Workload(5, 32768, 131, 16384, 5, "L R L^T, R symmetric partial permutation of rank 16384"),
}


def generate(w: Workload) -> np.ndarray:
    """Host generator: n x n uint64 residues."""
    out = np.zeros((w.n, w.n), np.uint64)
    _check(lib().ffb_generate_host(w.config, w.n, w.r, w.p, w.seed,
                                   out.ctypes.data_as(C.c_void_p)))
    return out


def generate_device(w: Workload, ctx=None):
    """Device generator: torch int32 tensor (n x n) of uint32 residues on the context device."""
    import torch

    from .ffldl import default_context
    ctx = ctx or default_context()
    a = torch.empty((w.n, w.n), dtype=torch.int32, device=f"cuda:{ctx.device}")
    _check(lib().ffb_generate_device(ctx.handle, w.config, w.n, w.r, w.p, w.seed, a.data_ptr()))
    return a


def config5_partners(w: Workload) -> np.ndarray:
    """partner[i] = j where the rank profile matrix R of config 5 has R(i, j) = 1, else -1."""
    out = np.zeros(w.n, np.int64)
    _check(lib().ffb_config5_partners(w.n, w.r, w.seed, out.ctypes.data_as(C.c_void_p)))
    return out
