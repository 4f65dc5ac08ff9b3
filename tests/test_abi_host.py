"""CPU-side checks of the C ABI: the library loads, exports every symbol include/dx.h declares,
host-side budget arithmetic agrees with the oracle, and the product never touches oracle/."""
import ctypes
import os
import re

import numpy as np

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    import __graft_entry__
    __graft_entry__.build()
    return ctypes.CDLL(os.path.join(ROOT, "paper_2511_15015_b200", "libdx.so"))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "dx.h")).read()
    names = set(re.findall(r"\b(dx_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 20
    lib = _lib()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2511_15015_b200 import dx
    assert set(dx.EXPORTED) <= names


def test_host_budget_arithmetic_matches_oracle():
    from paper_2511_15015_b200 import dx
    rng = np.random.default_rng(0)
    for H, I, g in [(64, 128, 32), (2048, 768, 128), (2048, 512, 128), (256, 192, 64)]:
        for bits in (16, 4, 2):
            assert dx.dx_slot_bytes(H, I, g, bits) == oracle.slot_bytes(H, I, g, bits)
    for _ in range(2000):
        N = int(rng.integers(1, 513)); Sl = int(rng.integers(1, 10**6)); Sh = Sl + int(rng.integers(1, 10**7))
        s = int(rng.integers(0, 3)); M = int(rng.integers(0, (N + 2) * Sh))
        assert dx.dx_solve_n_hot(M, N, Sh, Sl, s) == oracle.n_hot(M, N, Sh, Sl, s)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2511_15015_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
                assert "oracle.h" not in src and "_oracle.so" not in src, f
