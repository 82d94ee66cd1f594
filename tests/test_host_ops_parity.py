"""Byte-exact parity of the product's reference-surface host ops against the
oracle on identical bytes:

* fill_halo_clamped (workload.hpp:66-67) through imb_fill_halo_clamped vs the
  oracle's halo fill, on random padded fields of several shapes and halos;
* checksum (workload.hpp:82-85) through imb_checksum_padded (host) vs
  orc_checksum of the same interior bytes, and — on the GPU — the device
  team's imb_team_checksum vs orc_checksum of the downloaded slab.
"""
import ctypes as C

import numpy as np
import pytest

from paper_1507_01265_b200 import _lib
from paper_1507_01265_b200.mpdata import Options, Team

P64 = C.POINTER(C.c_double)
SHAPES = [(3, 3, 3, 1), (4, 5, 6, 1), (8, 9, 10, 2), (5, 3, 7, 3), (16, 4, 3, 2)]


def _padded(rng, n, m, l, h, special=False):
    a = rng.standard_normal((n + 2 * h, m + 2 * h, l + 2 * h))
    if special:  # signed zeros, subnormals, infinities: byte-level hashing must see them
        a.flat[::7] = -0.0
        a.flat[1::11] = 5e-324
        a.flat[2::13] = np.inf
    return np.ascontiguousarray(a)


@pytest.mark.parametrize("n,m,l,h", SHAPES)
@pytest.mark.parametrize("special", [False, True])
def test_fill_halo_clamped_matches_oracle_bytes(orc, n, m, l, h, special):
    rng = np.random.default_rng(n * 100 + m * 10 + l + h)
    f = _padded(rng, n, m, l, h, special)
    want = orc.fill_halo_clamped(f, n, m, l, h)
    got = f.copy()
    lib = _lib.load()
    d = _lib.imb_domain(n, m, l, h)
    _lib.check(lib.imb_fill_halo_clamped(C.byref(d), got.ctypes.data_as(P64)))
    assert got.tobytes() == want.tobytes()
    # interior untouched, every halo cell equals its clamped interior cell
    assert got[h:-h, h:-h, h:-h].tobytes() == f[h:-h, h:-h, h:-h].tobytes()
    ii = np.clip(np.arange(-h, n + h), 0, n - 1) + h
    jj = np.clip(np.arange(-h, m + h), 0, m - 1) + h
    kk = np.clip(np.arange(-h, l + h), 0, l - 1) + h
    assert got.tobytes() == f[np.ix_(ii, jj, kk)].tobytes()


@pytest.mark.parametrize("n,m,l,h", SHAPES)
@pytest.mark.parametrize("special", [False, True])
def test_checksum_padded_matches_oracle(orc, n, m, l, h, special):
    rng = np.random.default_rng(7 + n + m + l + h)
    f = _padded(rng, n, m, l, h, special)
    out = C.c_uint64()
    d = _lib.imb_domain(n, m, l, h)
    _lib.check(_lib.load().imb_checksum_padded(C.byref(d), f.ctypes.data_as(P64), C.byref(out)))
    interior = np.ascontiguousarray(f[h:-h, h:-h, h:-h])
    assert out.value == orc.checksum(interior)
    # the halo never enters the checksum
    g = f.copy()
    g[:h] = 123.0
    out2 = C.c_uint64()
    _lib.check(_lib.load().imb_checksum_padded(C.byref(d), g.ctypes.data_as(P64), C.byref(out2)))
    assert out2.value == out.value


def test_checksum_known_answers(orc):
    # FNV-1a 64 over the little-endian bytes: the empty
    # offset basis and one hand-computed value pin the byte order.
    assert orc.checksum(np.zeros(0)) == 0xCBF29CE484222325
    h = 0xCBF29CE484222325
    for b in np.array([1.0]).tobytes():
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    assert orc.checksum(np.array([1.0])) == h


@pytest.mark.gpu
@pytest.mark.parametrize("fp64", [True, False])
def test_team_checksum_matches_oracle_bytes(orc, fp64):
    opts = Options(2, True, fp64)
    with Team(20, 12, 32, opts, i0=0, ni=20) as t:
        t.init_recipe(2, 9)
        t.run(3)
        x = t.download("x")
        assert t.checksum() == orc.checksum(x)
