"""Pins the MPDATA oracle (oracle/mpdata_oracle.c) — CPU only.

The reference ships no MPDATA implementation or golden data,
so the oracle is pinned by: an independent numpy restatement, analytic
properties of the scheme (SURVEY.md §4 "How the new build should test"),
a hand-computed 1-D case, and self-generated golden checksums
(tests/golden/make_golden.py).
"""
import json
from pathlib import Path

import numpy as np
import pytest

from tests import np_mpdata

GOLDEN = Path(__file__).parent / "golden"

CASES = [(0, 1, False), (1, 2, False), (2, 2, True), (2, 3, True), (0, 2, True), (1, 3, False)]


@pytest.mark.parametrize("recipe,iord,nonos", CASES)
def test_matches_numpy_restatement(orc, recipe, iord, nonos):
    x, u, v, w, h = orc.init_fields(recipe, 12, 10, 8, seed=7)
    ref = x
    for _ in range(3):
        ref = np_mpdata.step(ref, u, v, w, h, iord=iord, nonos=nonos)
    got = orc.run(x, u, v, w, h, iord=iord, nonos=nonos, steps=3)
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("recipe,iord,nonos", CASES)
def test_mass_conservation(orc, recipe, iord, nonos):
    # Flux form + periodic boundaries: sum(h * psi) is invariant.
    x, u, v, w, h = orc.init_fields(recipe, 16, 12, 10, seed=3)
    m0 = float(np.sum(h * x))
    y = orc.run(x, u, v, w, h, iord=iord, nonos=nonos, steps=5)
    assert abs(float(np.sum(h * y)) - m0) <= 1e-12 * abs(m0)


@pytest.mark.parametrize("iord,nonos", [(1, False), (2, False), (2, True), (3, True)])
def test_constant_preserved_under_divergence_free_flow(orc, iord, nonos):
    # Solid-body rotation on the staggered grid is exactly divergence-free:
    # a constant field must stay constant bit-for-bit, for any density h.
    x, u, v, w, h = orc.init_fields(2, 16, 12, 10, seed=5)
    x[:] = 2.5
    y = orc.run(x, u, v, w, h, iord=iord, nonos=nonos, steps=4)
    assert np.all(y == 2.5)


def test_iord1_is_donor_cell(orc):
    x, u, v, w, h = orc.init_fields(0, 9, 8, 7, seed=11)
    got = orc.run(x, u, v, w, h, iord=1, nonos=False, steps=1)
    want = np_mpdata.update(x, u, v, w, h)
    np.testing.assert_array_equal(got, want)


def _mpdata_1d(psi, c, h, iord, eps=1e-15):
    """Hand-written scalar 1-D MPDATA (V = W = 0) for the reduction test."""
    n = len(psi)
    F = lambda a, b, cc: max(cc, 0.0) * a + min(cc, 0.0) * b  # noqa: E731

    def upd(x, vel):
        f = [F(x[(i - 1) % n], x[i], vel[i]) for i in range(n)]
        return [x[i] - (f[(i + 1) % n] - f[i]) / h[i] for i in range(n)]

    cur = upd(psi, c)
    vel = c
    for _ in range(2, iord + 1):
        nv = []
        for i in range(n):
            U = vel[i]
            hb = 0.5 * (h[(i - 1) % n] + h[i])
            a, b = abs(cur[i]), abs(cur[(i - 1) % n])
            A = (a - b) / ((a + b) + eps)
            nv.append((abs(U) - U * U / hb) * A)
        vel = nv
        cur = upd(cur, vel)
    return cur


@pytest.mark.parametrize("iord", [1, 2, 3])
def test_one_dimensional_reduction(orc, iord):
    n, m, l = 11, 4, 5
    rng = np.random.default_rng(1)
    psi = 1 + rng.random(n)
    c = rng.uniform(-0.4, 0.4, n)
    h = rng.uniform(0.8, 1.2, n)
    X = np.broadcast_to(psi[:, None, None], (n, m, l)).copy()
    U = np.broadcast_to(c[:, None, None], (n, m, l)).copy()
    H = np.broadcast_to(h[:, None, None], (n, m, l)).copy()
    Z = np.zeros((n, m, l))
    got = orc.run(X, U, Z, Z, H, iord=iord, nonos=False, steps=1)
    want = np.array(_mpdata_1d(list(psi), list(c), list(h), iord))
    for j in range(m):
        for k in range(l):
            np.testing.assert_allclose(got[:, j, k], want, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("iord", [2, 3])
def test_nonoscillatory_bounds(orc, iord):
    # Divergence-free flow with h = 1: the limited scheme creates no new
    # extrema, so the solution stays inside the initial [min, max] range.
    x, u, v, w, h = orc.init_fields(2, 24, 20, 16, seed=9)
    h[:] = 1.0
    lo, hi = x.min(), x.max()
    y = orc.run(x, u, v, w, h, iord=iord, nonos=True, steps=6)
    assert y.min() >= lo - 1e-12 and y.max() <= hi + 1e-12
    # ... while the unlimited scheme overshoots at the cube's discontinuity.
    z = orc.run(x, u, v, w, h, iord=iord, nonos=False, steps=6)
    assert z.max() > hi + 1e-6 or z.min() < lo - 1e-6


def test_thread_count_invariance(orc):
    # workload.hpp:130-131 / SPEC.md:297: the checksum never depends on threads.
    x, u, v, w, h = orc.init_fields(2, 16, 24, 8, seed=42)
    sums = {orc.checksum(orc.run(x, u, v, w, h, iord=2, nonos=True, steps=3, threads=t))
            for t in (1, 2, 3, 4, 7)}
    assert len(sums) == 1


def test_fp32_tracks_fp64(orc):
    x, u, v, w, h = orc.init_fields(2, 16, 12, 10, seed=2)
    xs = orc.init_fields(2, 16, 12, 10, seed=2, dtype=np.float32)
    y64 = orc.run(x, u, v, w, h, iord=2, nonos=True, steps=5)
    y32 = orc.run(*xs, iord=2, nonos=True, steps=5)
    np.testing.assert_allclose(y32, y64, rtol=2e-5, atol=2e-5)


def test_slab_init_is_slice_of_global(orc):
    # init is a pure function of the global index (workload.hpp:61-63), so a
    # slab (with wrapped halo planes) is a slice of the periodic global field.
    g = orc.init_fields(2, 20, 8, 6, seed=4)
    s = orc.init_fields(2, 20, 8, 6, seed=4, i0=-3, ni=26)
    for a, b in zip(g, s):
        np.testing.assert_array_equal(b, np.concatenate([a[-3:], a, a[:3]]))


def test_stage_max7_matches_naive(orc):
    # SPEC.md:298 / :488: max7 vs a naive evaluation on random 8^3 fields.
    rng = np.random.default_rng(0)
    n = m = l = 8
    hal = 1
    for _ in range(10):
        f = rng.random((n + 2, m + 2, l + 2))
        f = orc.fill_halo_clamped(f, n, m, l, hal)
        mx = orc.stage7(f, n, m, l, hal, True)
        mn = orc.stage7(f, n, m, l, hal, False)
        for i in range(1, n + 1):
            for j in range(1, m + 1):
                for k in range(1, l + 1):
                    nb = [f[i, j, k], f[i - 1, j, k], f[i + 1, j, k], f[i, j - 1, k],
                          f[i, j + 1, k], f[i, j, k - 1], f[i, j, k + 1]]
                    assert mx[i, j, k] == max(nb) and mn[i, j, k] == min(nb)


def test_golden_checksums(orc):
    rows = json.loads((GOLDEN / "mpdata_checksums.json").read_text())
    assert rows
    for r in rows:
        dt = np.float64 if r["precision"] == "fp64" else np.float32
        f = orc.init_fields(r["recipe"], *r["grid"], seed=r["seed"], dtype=dt)
        y = orc.run(*f, iord=r["iord"], nonos=r["nonos"], steps=r["steps"], threads=2)
        assert f"{orc.checksum(y):016x}" == r["checksum"], r
