"""MPDATA pinned by properties of the published scheme rather than by a
second transcription of it (the oracle, tests/np_mpdata.py and
the golden checksums all come from one reading of SURVEY.md App. A).

The reference ships no MPDATA, so parity stays "unpinned by
the reference"; these tests pin the oracle — and through the GPU parity
tests the product — to what the literature proves about the scheme
(Smolarkiewicz 1984, J. Comput. Phys. 54; Smolarkiewicz & Margolin 1998):

* donor cell (IORD=1) is first-order accurate, MPDATA with one corrective
  pass (IORD=2) is second-order accurate for constant flow: on grid
  refinement at fixed Courant number and physical time the error of a
  smooth profile falls ~2x (IORD=1) and ~4x (IORD=2). A wrong sign or
  factor in the antidiffusive velocity (|U| - U^2/h) A breaks the 4x;
* the transverse (cross) terms 0.125 U (V-sum) B / h of the 3-D
  pseudo-velocity are what keep the scheme second order for flow that is
  not aligned with the grid: a diagonal 2-D advection converges at ~4x with
  them; dropping them (here: a restatement without cross terms) is first
  order and at this Courant number unstable, which shows the test sees
  those terms; a second corrective pass (IORD=3) raises the order further;
* the nonoscillatory option keeps a positive field inside the bounds of its
  initial values (monotone) and keeps the second-order convergence.

Small periodic grids with the inert extents at 3 cells, oracle on the CPU.
"""
import math

import numpy as np
import pytest

from tests import np_mpdata as npm

C_NUM = 0.25  # Courant number along each active axis


def advect_1d(orc, n, iord, nonos=False, cross=True):
    """psi = 2 + sin(2 pi x / n) advected for one full period along i."""
    x = (np.arange(n) + 0.5) / n
    prof = 2.0 + np.sin(2 * np.pi * x)
    shape = (n, 3, 3)
    psi = np.broadcast_to(prof[:, None, None], shape).copy()
    u = np.full(shape, C_NUM)
    z = np.zeros(shape)
    h = np.ones(shape)
    steps = int(round(n / C_NUM))
    out = orc.run(psi, u, z, z, h, iord=iord, nonos=nonos, steps=steps, threads=2)
    return float(np.sqrt(np.mean((out - psi) ** 2)))


def advect_diag(orc, n, iord, nonos=False, cross=True):
    """psi = 2 + sin(2 pi (x + y) / n) advected along the diagonal u = v for one period."""
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    prof = 2.0 + np.sin(2 * np.pi * (i + j + 1.0) / n)
    shape = (n, n, 3)
    psi = np.broadcast_to(prof[:, :, None], shape).copy()
    u = np.full(shape, C_NUM)
    v = np.full(shape, C_NUM)
    z = np.zeros(shape)
    h = np.ones(shape)
    steps = int(round(n / C_NUM))
    if cross:
        out = orc.run(psi, u, v, z, h, iord=iord, nonos=nonos, steps=steps, threads=2)
    else:
        out = psi.copy()
        for _ in range(steps):
            out = _step_without_cross_terms(out, u, v, z, h)
    return float(np.sqrt(np.mean((out - psi) ** 2)))


def _step_without_cross_terms(x, U, V, W, h):
    """IORD=2 with the pseudo-velocities' transverse terms removed (a
    deliberately wrong scheme: shows the diagonal test detects them)."""
    x1 = npm.update(x, U, V, W, h)
    a = np.abs(x1)
    eps = npm.EPS

    def face(vel, axis):
        aL = npm.sh(a, -1, axis)
        hb = 0.5 * (npm.sh(h, -1, axis) + h)
        return (np.abs(vel) - vel * vel / hb) * (a - aL) / (a + aL + eps)

    return npm.update(x1, face(U, 0), face(V, 1), face(W, 2), h)


def orders(errs):
    return [math.log2(errs[q] / errs[q + 1]) for q in range(len(errs) - 1)]


def test_donor_cell_is_first_order(orc):
    e = [advect_1d(orc, n, 1) for n in (32, 64, 128)]
    o = orders(e)
    assert all(0.8 < q < 1.2 for q in o), (e, o)


@pytest.mark.parametrize("iord", [2, 3])
def test_mpdata_is_second_order_1d(orc, iord):
    e = [advect_1d(orc, n, iord) for n in (32, 64, 128)]
    o = orders(e)
    assert all(q > 1.8 for q in o), (e, o)
    assert e[-1] < 0.05 * advect_1d(orc, 128, 1)  # far below donor cell's error


def test_cross_terms_keep_second_order_on_the_diagonal(orc):
    with_c = [advect_diag(orc, n, 2) for n in (32, 64, 128)]
    o = orders(with_c)
    assert all(q > 1.85 for q in o), (with_c, o)
    # the same scheme without the transverse terms is not second order (at
    # C = 0.25 on the diagonal it is not even stable)
    without = [advect_diag(orc, n, 2, cross=False) for n in (32, 64, 128)]
    assert orders(without)[0] < 1.2 and without[-1] > 10 * with_c[-1], without


def test_second_corrective_pass_raises_the_order_on_the_diagonal(orc):
    # IORD=3 (config 5's scheme): a third pass on the corrected field cancels
    # the next error term for constant flow (~3rd order here)
    e = [advect_diag(orc, n, 3) for n in (32, 64, 128)]
    o = orders(e)
    assert all(q > 2.5 for q in o), (e, o)


def test_nonoscillatory_keeps_bounds_and_order(orc):
    e = [advect_1d(orc, n, 2, nonos=True) for n in (32, 64, 128)]
    o = orders(e)
    assert o[-1] > 1.6, (e, o)  # the limiter clips the extrema a little, still ~2nd order
    # monotone on a square wave: stays inside [1, 3] of the initial field
    n = 64
    prof = np.where((np.arange(n) >= 16) & (np.arange(n) < 32), 3.0, 1.0)
    shape = (n, 3, 3)
    psi = np.broadcast_to(prof[:, None, None], shape).copy()
    u = np.full(shape, C_NUM)
    z = np.zeros(shape)
    out = orc.run(psi, u, z, z, np.ones(shape), iord=2, nonos=True, steps=100, threads=2)
    assert out.min() >= 1.0 - 1e-12 and out.max() <= 3.0 + 1e-12
    plain = orc.run(psi, u, z, z, np.ones(shape), iord=2, nonos=False, steps=100, threads=2)
    assert plain.max() > 3.0 + 1e-6 or plain.min() < 1.0 - 1e-6  # the limiter is doing work


@pytest.mark.gpu
@pytest.mark.parametrize("fp64", [True, False])
def test_product_converges_at_second_order_on_the_diagonal(fp64):
    # The same property through the product (fused kernel: l = 32).
    from paper_1507_01265_b200.mpdata import Options, Team
    dt = np.float64 if fp64 else np.float32
    errs = []
    for n in (32, 64, 128):
        i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        prof = 2.0 + np.sin(2 * np.pi * (i + j + 1.0) / n)
        shape = (n, n, 32)
        psi = np.broadcast_to(prof[:, :, None], shape).astype(dt)
        u = np.full(shape, C_NUM, dt)
        z = np.zeros(shape, dt)
        with Team(*shape, Options(2, True, fp64)) as t:
            t.upload_all(psi, u, u, z, np.ones(shape, dt))
            t.run(int(round(n / C_NUM)))
            out = t.download("x").astype(np.float64)
        errs.append(float(np.sqrt(np.mean((out - psi) ** 2))))
    assert all(q > 1.8 for q in orders(errs)), errs
