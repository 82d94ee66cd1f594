"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle on the
same seeded inputs (BASELINE.json north_star tolerance: max relative error
1e-12 in fp64, 1e-5 in fp32; relative error floored at |ref| >= 1 per
SURVEY.md App. C #7), plus size-independent properties at full size."""
import numpy as np
import pytest

from paper_1507_01265_b200 import _lib, mpdata
from paper_1507_01265_b200.mpdata import Group, Options, Team

pytestmark = pytest.mark.gpu

TOL = {True: 1e-12, False: 1e-5}


def rel_err(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)) /
                        np.maximum(np.abs(b.astype(np.float64)), 1.0)))


def gpu_run(fields, opts, steps):
    n, m, l = fields[0].shape
    with Team(n, m, l, opts) as t:
        t.upload_all(*fields)
        t.run(steps)
        assert t.launches > 0
        return t.download("x")


def oracle_run(orc, fields, opts, steps):
    return orc.run(*fields, iord=opts.iord, nonos=opts.nonos, steps=steps, threads=8)


def test_config1_parity(orc):
    # BASELINE config 1: 64x64x32 fp64, periodic, 10 steps, IORD=2, nonos off.
    opts = Options(iord=2, nonos=False, fp64=True)
    f = orc.init_fields(1, 64, 64, 32, seed=42)
    got = gpu_run(f, opts, 10)
    want = oracle_run(orc, f, opts, 10)
    assert rel_err(got, want) <= 1e-12
    assert want.min() < 1.5  # the divergent config exercises |psi| ratios


def test_config2_parity(orc):
    # BASELINE config 2: 256x256x64 fp64, 50 steps, IORD=2, limiter on.
    opts = Options(iord=2, nonos=True, fp64=True)
    f = orc.init_fields(2, 256, 256, 64, seed=42)
    got = gpu_run(f, opts, 50)
    want = oracle_run(orc, f, opts, 50)
    assert rel_err(got, want) <= 1e-12


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("iord,nonos", [(1, False), (2, False), (2, True), (3, True), (3, False),
                                        (4, True), (4, False)])
@pytest.mark.parametrize("recipe", [0, 2])
def test_scheme_matrix_parity(orc, fp64, iord, nonos, recipe):
    opts = Options(iord=iord, nonos=nonos, fp64=fp64)
    dt = np.float64 if fp64 else np.float32
    f = orc.init_fields(recipe, 24, 20, 36, seed=5, dtype=dt)
    got = gpu_run(f, opts, 4)
    want = oracle_run(orc, f, opts, 4)
    assert rel_err(got, want) <= TOL[fp64]


@pytest.mark.parametrize("shape", [(5, 3, 3), (7, 33, 65), (16, 129, 20), (40, 8, 256)])
def test_ragged_shapes_parity(orc, shape):
    opts = Options(iord=3, nonos=True, fp64=True)
    f = orc.init_fields(0, *shape, seed=17)
    got = gpu_run(f, opts, 3)
    want = oracle_run(orc, f, opts, 3)
    assert rel_err(got, want) <= 1e-12


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("recipe", [0, 2])
def test_device_init_is_bit_identical_to_host(orc, fp64, recipe):
    dt = np.float64 if fp64 else np.float32
    n, m, l = 20, 12, 10
    want = orc.init_fields(recipe, n, m, l, seed=99, dtype=dt)
    with Team(n, m, l, Options(fp64=fp64), i0=6, ni=9) as t:
        t.init_recipe(recipe, 99)
        for name, ref in zip("xuvwh", want):
            np.testing.assert_array_equal(t.download(name), ref[6:15])


@pytest.mark.parametrize("shares", [[16, 16], [10, 6, 16], [3, 29], [8, 8, 8, 8], [11, 21]])
@pytest.mark.parametrize("opts", [Options(2, True, True), Options(3, True, False),
                                  Options(2, False, True)])
def test_group_decomposition_is_bit_identical(shares, opts):
    # P slabs on one GPU exchanging halos by device copies must reproduce the
    # single-slab result exactly: the per-cell arithmetic is identical, so
    # any difference is a halo/indexing bug.
    n, m, l = sum(shares), 24, 40
    R = mpdata.step_radius(opts)
    if min(shares) < R:
        pytest.skip("slab thinner than the step radius")
    with Team(n, m, l, opts) as t:
        t.init_recipe(2, 7)
        t.run(5)
        single = t.download("x")
    g = Group(n, m, l, shares, opts=opts)
    g.init_recipe(2, 7)
    per, wall = g.run(5)
    assert len(per) == len(shares) and wall > 0
    np.testing.assert_array_equal(g.download("x"), single)
    g.close()


@pytest.mark.parametrize("shares", [[32], [16, 16], [9, 7, 16], [8, 8, 8, 8]])
@pytest.mark.parametrize("opts", [Options(2, True, True), Options(2, False, False),
                                  Options(3, True, True)])
def test_group_flag_sync_is_bit_identical(shares, opts):
    # Flag-synchronised ring (cuStreamWaitValue64 / WriteValue64 on device
    # flag words, halos pushed by the step kernel): same bits as one slab.
    n, m, l = sum(shares), 20, 64
    with Team(n, m, l, opts) as t:
        t.init_recipe(2, 11)
        t.run(6)
        single = t.download("x")
    g = Group(n, m, l, shares, opts=opts)
    g.set_sync("flags")
    g.init_recipe(2, 11)
    g.run(2)
    g.run(4)  # continues in flag mode across calls
    np.testing.assert_array_equal(g.download("x"), single)
    g.close()


@pytest.mark.timeout(120)
@pytest.mark.parametrize("shares", [[16, 16], [9, 7, 16]])
def test_group_sync_mode_switching_is_bit_identical(shares):
    # events -> flags -> events -> flags must neither deadlock (the
    # flag words are kept in step by every event step) nor change a bit.
    opts = Options(2, True, True)
    n, m, l = sum(shares), 20, 64
    with Team(n, m, l, opts) as t:
        t.init_recipe(2, 11)
        t.run(9)
        single = t.download("x")
    g = Group(n, m, l, shares, opts=opts)
    g.init_recipe(2, 11)
    g.run(2)  # events
    g.set_sync("flags")
    g.run(3)
    g.set_sync("events")
    g.run(2)
    g.set_sync("flags")
    g.run(2)
    np.testing.assert_array_equal(g.download("x"), single)
    g.close()


def test_step_host_rejects_bad_buffers():
    # the C side copies ni*m*l elements each way, so the mirror
    # must refuse wrong dtypes, shapes and non-contiguous or read-only outputs.
    with Team(16, 8, 32, Options(2, True, True)) as t:
        t.init_recipe(2, 1)
        good = np.zeros(t.shape)
        with pytest.raises(_lib.ContractError):
            t.step_host(np.zeros((15, 8, 32)), good)
        with pytest.raises(_lib.ContractError):
            t.step_host(good, np.zeros(t.shape, dtype=np.float32))
        with pytest.raises(_lib.ContractError):
            t.step_host(good, np.zeros((16, 8, 64))[:, :, ::2])
        ro = np.zeros(t.shape)
        ro.flags.writeable = False
        with pytest.raises(_lib.ContractError):
            t.step_host(good, ro)
        out = np.zeros(t.shape)
        t.step_host(good.astype(np.float32), out)  # inputs are converted


def test_group_with_uploaded_fields(orc):
    opts = Options(2, True, True)
    f = orc.init_fields(0, 30, 16, 24, seed=3)
    g = Group(30, 16, 24, [12, 18], opts=opts)
    off = 0
    for t in g.teams:
        t.upload_all(*(a[off:off + t.ni] for a in f))
        off += t.ni
    g.run(3)
    want = oracle_run(orc, f, opts, 3)
    assert rel_err(g.download("x"), want) <= 1e-12
    g.close()


def test_step_host_matches_run_and_reset(orc):
    opts = Options(2, True, True)
    f = orc.init_fields(2, 32, 24, 16, seed=1)
    with Team(32, 24, 16, opts) as t:
        t.upload_all(*f)
        xin = np.ascontiguousarray(f[0])
        xout = np.empty_like(xin)
        t.step_host(xin, xout)
        t.reset()
        t.run(1)
        np.testing.assert_array_equal(t.download("x"), xout)
        c1 = t.checksum()
        t.reset()
        t.run(1)
        assert t.checksum() == c1
    assert rel_err(xout, oracle_run(orc, f, opts, 1)) <= 1e-12


@pytest.mark.parametrize("opts,shape", [(Options(2, True, True), (96, 20, 64)),
                                        (Options(2, False, False), (64, 7, 128)),
                                        (Options(2, True, False), (200, 13, 32)),
                                        (Options(2, True, True), (400, 6, 32))])  # 16 chunks
def test_pipelined_step_host_is_bit_identical(orc, opts, shape):
    # step_host on a fused shape takes the chunked H2D / kernel / D2H pipeline;
    # it must equal the device-resident run() bit for bit.
    dt = np.float64 if opts.fp64 else np.float32
    f = orc.init_fields(2, *shape, seed=31, dtype=dt)
    with Team(*shape, opts) as t:
        t.upload_all(*f)
        xin = np.ascontiguousarray(f[0])
        xout = np.empty_like(xin)
        t.step_host(xin, xout)
        xout2 = np.empty_like(xin)
        t.step_host(xout, xout2)  # second step from the host result
        t.reset()
        t.run(2)
        np.testing.assert_array_equal(t.download("x"), xout2)
    assert rel_err(xout2, oracle_run(orc, f, opts, 2)) <= TOL[opts.fp64]


def test_stage_max7_min7_on_gpu(orc):
    import ctypes as C
    n, m, l, h = 8, 9, 10, 1
    rng = np.random.default_rng(3)
    f = orc.fill_halo_clamped(rng.random((n + 2, m + 2, l + 2)), n, m, l, h)
    lib = _lib.load()
    d = _lib.imb_domain(n, m, l, h)
    P = C.POINTER(C.c_double)
    for is_max, fn in ((True, lib.imb_stage_max7), (False, lib.imb_stage_min7)):
        out = np.zeros_like(f)
        _lib.check(fn(C.byref(d), f.ctypes.data_as(P), out.ctypes.data_as(P)))
        want = orc.stage7(f, n, m, l, h, is_max)
        np.testing.assert_array_equal(out[1:-1, 1:-1, 1:-1], want[1:-1, 1:-1, 1:-1])


def test_contract_errors_on_gpu():
    with pytest.raises(_lib.ContractError):
        Team(16, 8, 8, Options(3, True), i0=0, ni=4)  # slab thinner than R=5
    with pytest.raises(_lib.ContractError):
        Group(16, 8, 8, [8, 7])  # shares must sum to n
    with pytest.raises(_lib.ConfigError):
        Team(16, 8, 8, Options(2, True), device=64)
    with Team(16, 8, 8) as t:
        with pytest.raises(_lib.ContractError):
            t.upload("x", np.zeros((15, 8, 8)))


def test_ipc_export_and_connect_contracts():
    # The cross-process NVLink push path (imb_team_connect_ipc) needs one GPU
    # per rank, so only its blob format and argument checks run here; its
    # push + flag protocol is the one test_group_flag_sync_is_bit_identical
    # exercises in-process.
    with Team(32, 16, 64) as a, Team(32, 16, 32) as b:
        a.init_recipe(2, 42)
        blob = a.ipc_export()
        assert len(blob) == 512 and int.from_bytes(blob[:4], "little") == 0x1B200C0D
        with pytest.raises(_lib.ContractError):
            a.connect_ipc(b"\0" * 512, b"\0" * 512, 2, 0)  # not a blob
        with pytest.raises(_lib.ContractError):
            a.connect_ipc(b.ipc_export(), b.ipc_export(), 2, 0)  # plane size differs
        with pytest.raises(_lib.ContractError):
            a.connect_ipc(blob, blob, 2, 2)  # rank out of range
        a.connect_ipc(blob, blob, 1, 0)  # single rank: periodic self push, no mapping
        a.run(2)
        with Team(32, 16, 64) as c:
            c.init_recipe(2, 42)
            c.run(2)
            np.testing.assert_array_equal(a.download("x"), c.download("x"))
    with Team(32, 16, 64, Options(3, False)) as s:  # staged scheme: no fused push
        with pytest.raises(_lib.ConfigError):
            s.ipc_export()


def _mass(h, x):
    # plane-chunked pairwise sums, combined exactly (fsum): no 2 GB temporaries
    import math
    return math.fsum(float(np.sum(h[i:i + 64].astype(np.float64) * x[i:i + 64]))
                     for i in range(0, x.shape[0], 64))


@pytest.mark.parametrize("fp64", [True, False])
def test_full_size_properties_c5(fp64):
    # BASELINE config 5 grid (2048x1024x128, IORD=3 + limiter): the largest
    # single-GPU problem; mass conservation and bounds after 2 steps.
    opts = Options(3, True, fp64)
    with Team(2048, 1024, 128, opts) as t:
        t.init_recipe(2, 42)
        x0 = t.download("x")
        h = t.download("h")
        m0 = _mass(h, x0.astype(np.float64))
        lo, hi = float(x0.min()), float(x0.max())
        del x0
        t.run(2)
        x = t.download("x").astype(np.float64)
    tol = 1e-12 if fp64 else 1e-5
    assert abs(_mass(h, x) - m0) <= tol * m0
    assert x.min() >= lo - 1e-3 and x.max() <= hi + 1e-3


@pytest.mark.parametrize("fp64", [True, False])
def test_full_size_properties(fp64):
    # BASELINE config 4 grid (1024x512x128): mass conservation and the
    # limiter's bounds hold at full size (size-independent parity checks).
    opts = Options(2, True, fp64)
    with Team(1024, 512, 128, opts) as t:
        t.init_recipe(2, 42)
        x0 = t.download("x").astype(np.float64)
        h = t.download("h").astype(np.float64)
        m0 = float(np.sum(h * x0))
        t.run(3)
        x = t.download("x").astype(np.float64)
    tol = 1e-12 if fp64 else 1e-5
    assert abs(float(np.sum(h * x)) - m0) <= tol * m0
    assert x.min() >= x0.min() - 1e-3 and x.max() <= x0.max() + 1e-3


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("nonos", [True, False])
@pytest.mark.parametrize("shape", [(6, 5, 32), (17, 13, 64), (12, 40, 128), (9, 3, 128),
                                   (30, 29, 32)])
def test_fused_kernel_parity(orc, fp64, nonos, shape):
    # Shapes with l in {32, 64, 128} take the fused streaming kernel; m not a
    # multiple of the j-tile and m smaller than the tile exercise the wrap.
    opts = Options(iord=2, nonos=nonos, fp64=fp64)
    dt = np.float64 if fp64 else np.float32
    f = orc.init_fields(2 if nonos else 1, *shape, seed=23, dtype=dt)
    got = gpu_run(f, opts, 3)
    want = oracle_run(orc, f, opts, 3)
    assert rel_err(got, want) <= TOL[fp64]


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("shape", [(12, 5, 32), (17, 13, 64), (20, 40, 128), (11, 3, 128)])
def test_fused_iord3_parity(orc, fp64, shape):
    # BASELINE config 5's scheme (IORD=3 + limiter) through the two fused
    # launches (pass 2 writing limited velocities and bounds, then pass 3).
    opts = Options(iord=3, nonos=True, fp64=fp64)
    dt = np.float64 if fp64 else np.float32
    f = orc.init_fields(2, *shape, seed=29, dtype=dt)
    got = gpu_run(f, opts, 3)
    want = oracle_run(orc, f, opts, 3)
    assert rel_err(got, want) <= TOL[fp64]


@pytest.mark.parametrize("shares", [[16, 16], [9, 7, 16], [6, 26], [8, 8, 8, 8]])
@pytest.mark.parametrize("opts", [Options(2, True, True), Options(2, False, False),
                                  Options(3, True, True)])
def test_group_decomposition_fused_is_bit_identical(shares, opts):
    n, m, l = sum(shares), 20, 64
    with Team(n, m, l, opts) as t:
        t.init_recipe(2, 7)
        t.run(4)
        single = t.download("x")
    g = Group(n, m, l, shares, opts=opts)
    g.init_recipe(2, 7)
    g.run(4)
    np.testing.assert_array_equal(g.download("x"), single)
    g.close()


@pytest.mark.parametrize("shape", [(5, 18, 128), (7, 19, 128), (5, 20, 128), (7, 21, 128),
                                   (16, 47, 128), (6, 130, 128)])
@pytest.mark.parametrize("iord", [2, 3])
def test_fp32_staged_inputs_parity(orc, shape, iord):
    # fp32 at l = 128 stages psi^n and h in shared memory with bulk async copies
    # (rings refilled one iteration ahead): with the extra halo rows (18 region
    # rows) m = 20 is the smallest staged tile (rows -1..18 without repeats) and
    # m = 18, 19 take the unstaged kernel; short slabs give one- and two-plane
    # segments, m = 130 wraps the last tile's rows.
    opts = Options(iord=iord, nonos=True, fp64=False)
    f = orc.init_fields(2, *shape, seed=31, dtype=np.float32)
    got = gpu_run(f, opts, 3)
    want = oracle_run(orc, f, opts, 3)
    assert rel_err(got, want) <= TOL[False]


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("shape", [(8, 14, 128), (9, 15, 128), (7, 17, 128), (8, 18, 128),
                                   (6, 28, 128), (6, 29, 128), (5, 43, 128)])
def test_extra_row_tiles_parity(orc, fp64, shape):
    # l = 128 with the limiter runs 18 region rows on 16 warps (14 output rows
    # per tile; warps 0 and 15 also handle the outermost halo rows): m equal
    # to, one above, and a little beyond one or two tiles, and m below the 18
    # region rows (the tile's rows wrap around j).
    opts = Options(iord=2, nonos=True, fp64=fp64)
    dt = np.float64 if fp64 else np.float32
    f = orc.init_fields(2, *shape, seed=37, dtype=dt)
    got = gpu_run(f, opts, 4)
    want = oracle_run(orc, f, opts, 4)
    assert rel_err(got, want) <= TOL[fp64]


@pytest.mark.parametrize("shares", [[9, 7, 16], [8, 8, 8, 8]])
@pytest.mark.parametrize("iord", [2, 3])
def test_group_extra_rows_fp64_is_bit_identical(shares, iord):
    # the fp64 l = 128 tiles (extra rows, TMEM rings) under slab decomposition
    opts = Options(iord, True, True)
    n, m, l = sum(shares), 31, 128
    with Team(n, m, l, opts) as t:
        t.init_recipe(2, 3)
        t.run(3)
        single = t.download("x")
    g = Group(n, m, l, shares, opts=opts)
    g.init_recipe(2, 3)
    g.run(3)
    np.testing.assert_array_equal(g.download("x"), single)
    g.close()


@pytest.mark.parametrize("shares", [[3, 4, 5], [8, 8], [3, 3, 3, 3]])
def test_group_fp32_staged_is_bit_identical(shares):
    opts = Options(2, True, False)
    n, m, l = sum(shares), 21, 128
    with Team(n, m, l, opts) as t:
        t.init_recipe(2, 5)
        t.run(3)
        single = t.download("x")
    g = Group(n, m, l, shares, opts=opts)
    g.init_recipe(2, 5)
    g.run(3)
    np.testing.assert_array_equal(g.download("x"), single)
    g.close()
