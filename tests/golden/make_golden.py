"""Regenerate tests/golden/ref_outputs.npz from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libffldl_ref.so, i.e.
/root/reference present at build time):  python tests/golden/make_golden.py

Every case is factored by the reference's own ffldl::ldlt through
oracle/ref_capi.cpp; inputs are regenerated from their seeds by the tests
(configs via ffb_generate_host, the rest via numpy's PCG64), so only outputs
and an input checksum are stored.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.bind import Checker  # noqa: E402
from golden_cases import golden_cases  # noqa: E402


def main():
    ref = Checker("ref")
    out = {}
    for name, p, a, variant, T in golden_cases():
        f = ref.ldlt(p, a, variant, T)
        out[f"{name}/sha"] = np.frombuffer(hashlib.sha256(a.tobytes()).digest(), np.uint8)
        out[f"{name}/perm"] = f.perm.astype(np.int32)
        out[f"{name}/lower"] = f.lower.astype(np.uint32)
        out[f"{name}/dkind"] = f.dkind.astype(np.int8)
        out[f"{name}/dval"] = f.dval.astype(np.uint32)
        out[f"{name}/dval2"] = f.dval2.astype(np.uint32)
        out[f"{name}/rank"] = np.array([f.rank], np.int64)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_outputs.npz")
    np.savez_compressed(path, **out)
    print(path, len(out) // 7, "cases", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
