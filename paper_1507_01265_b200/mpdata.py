"""Python mirror of the MPDATA workload API over the C-ABI.

``Team`` is the B200 ``TeamRunner`` (/root/reference/proj/include/imbalance/
workload.hpp:94-122): one GPU advancing one i-slab of a periodic global grid.
``Group`` is a ring of teams in one process (one host thread drives several
devices, or several slabs share one device for decomposition tests).
Host arrays are numpy arrays of shape (ni, m, l) in the team precision.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, imb_domain, imb_opts, load

FP64, FP32 = 0, 1
RECIPE_UNIFORM, RECIPE_GAUSS, RECIPE_ROTCUBE = 0, 1, 2
FIELDS = {"x": 0, "u": 1, "v": 2, "w": 3, "h": 4}


@dataclass(frozen=True)
class Options:
    iord: int = 2
    nonos: bool = True
    fp64: bool = True

    def c(self) -> imb_opts:
        return imb_opts(self.iord, int(self.nonos), FP64 if self.fp64 else FP32)

    @property
    def dtype(self):
        return np.float64 if self.fp64 else np.float32


def step_radius(opts: Options) -> int:
    r = load().imb_step_radius(C.byref(opts.c()))
    if r < 0:
        check(-r)
    return r


def _field_id(field) -> int:
    return FIELDS[field] if isinstance(field, str) else int(field)


class Team:
    """One GPU, one slab [i0, i0+ni) of the n x m x l periodic grid."""

    def __init__(self, n, m, l, opts: Options = Options(), device: int = 0, i0: int = 0,
                 ni: int | None = None, _handle=None):
        self.n, self.m, self.l = int(n), int(m), int(l)
        self.opts = opts
        self.i0 = int(i0)
        self.ni = int(n if ni is None else ni)
        self._owned = _handle is None
        if _handle is None:
            h = C.c_void_p()
            dom = imb_domain(self.n, self.m, self.l, 1)
            check(load().imb_team_create(C.byref(dom), C.byref(opts.c()), int(device), self.i0,
                                         self.ni, C.byref(h)))
            self._h = h
        else:
            self._h = _handle

    # -- lifetime ---------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) and self._owned:
            load().imb_team_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- fields -----------------------------------------------------------------
    @property
    def shape(self):
        return (self.ni, self.m, self.l)

    def init_recipe(self, recipe: int = RECIPE_ROTCUBE, seed: int = 42):
        check(load().imb_team_init_recipe(self._h, int(recipe), C.c_uint64(seed)))

    def upload(self, field, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=self.opts.dtype)
        if a.shape != self.shape:
            raise _lib.ContractError(f"upload shape {a.shape} != slab {self.shape}")
        check(load().imb_team_upload(self._h, _field_id(field), a.ctypes.data, a.nbytes))

    def upload_all(self, x, u, v, w, h):
        for name, a in zip("xuvwh", (x, u, v, w, h)):
            self.upload(name, a)

    def download(self, field="x") -> np.ndarray:
        out = np.empty(self.shape, dtype=self.opts.dtype)
        check(load().imb_team_download(self._h, _field_id(field), out.ctypes.data, out.nbytes))
        return out

    def reset(self):
        check(load().imb_team_reset(self._h))

    # -- stepping ---------------------------------------------------------------
    def run(self, steps: int):
        """Returns (compute seconds, wall seconds) measured with CUDA events."""
        comp, wall = C.c_double(), C.c_double()
        check(load().imb_team_run(self._h, int(steps), C.byref(comp), C.byref(wall)))
        return comp.value, wall.value

    def step_host(self, x_in: np.ndarray, x_out: np.ndarray):
        """One step from host buffers: x_in -> device -> step -> x_out. Both
        must be slab-shaped; x_out must be a writeable C-contiguous array of
        the team precision (the C side copies ni*m*l elements each way)."""
        a = np.ascontiguousarray(x_in, dtype=self.opts.dtype)
        if a.shape != self.shape:
            raise _lib.ContractError(f"step_host input shape {a.shape} != slab {self.shape}")
        if (not isinstance(x_out, np.ndarray) or x_out.shape != self.shape
                or x_out.dtype != self.opts.dtype or not x_out.flags.c_contiguous
                or not x_out.flags.writeable):
            raise _lib.ContractError(
                f"step_host output must be a writeable C-contiguous {np.dtype(self.opts.dtype)} "
                f"array of shape {self.shape}")
        check(load().imb_team_step_host(self._h, a.ctypes.data, x_out.ctypes.data))

    def checksum(self) -> int:
        out = C.c_uint64()
        check(load().imb_team_checksum(self._h, C.byref(out)))
        return out.value

    @property
    def launches(self) -> int:
        return int(load().imb_team_launch_count(self._h))

    def connect_nccl(self, uid: bytes, nranks: int, rank: int):
        check(load().imb_team_connect_nccl(self._h, uid, int(nranks), int(rank)))

    def ipc_export(self) -> bytes:
        buf = C.create_string_buffer(512)
        check(load().imb_team_ipc_export(self._h, buf))
        return buf.raw

    def connect_ipc(self, left: bytes, right: bytes, nranks: int, rank: int):
        check(load().imb_team_connect_ipc(self._h, left, right, int(nranks), int(rank)))


def ring_plan(rank: int, nranks: int, ni: int, R: int):
    """The per-step halo-swap plan the NCCL exchange executes:
    [(kind 'send'|'recv', peer, first_plane, planes)] in issue order."""
    kinds, peers = (C.c_int * 4)(), (C.c_int * 4)()
    first, planes = (C.c_int64 * 4)(), (C.c_int64 * 4)()
    check(load().imb_ring_plan(int(rank), int(nranks), int(ni), int(R), kinds, peers, first,
                               planes))
    return [("send" if kinds[q] == 0 else "recv", peers[q], first[q], planes[q]) for q in range(4)]


def slab_offsets(shares) -> list:
    arr = (C.c_int64 * max(len(shares), 1))(*shares)
    out = (C.c_int64 * max(len(shares), 1))()
    check(load().imb_slab_offsets(arr, len(shares), out))
    return list(out[:len(shares)])


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(load().imb_nccl_unique_id(buf))
    return buf.raw


class Group:
    """In-process ring of teams; slab g = [sum(shares[:g]), +shares[g])."""

    def __init__(self, n, m, l, shares, devices=None, opts: Options = Options()):
        self.n, self.m, self.l = int(n), int(m), int(l)
        self.shares = [int(s) for s in shares]
        devs = list(devices) if devices is not None else [0] * len(self.shares)
        self.opts = opts
        h = C.c_void_p()
        dom = imb_domain(self.n, self.m, self.l, 1)
        check(load().imb_group_create(C.byref(dom), C.byref(opts.c()), len(self.shares),
                                      (C.c_int * len(devs))(*devs),
                                      (C.c_int64 * len(self.shares))(*self.shares), C.byref(h)))
        self._h = h
        self.teams = []
        off = 0
        for g, s in enumerate(self.shares):
            th = C.c_void_p()
            check(load().imb_group_team(self._h, g, C.byref(th)))
            self.teams.append(Team(n, m, l, opts, devs[g], off, s, _handle=th))
            off += s

    def close(self):
        if getattr(self, "_h", None):
            for t in self.teams:
                t._h = None
            load().imb_group_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init_recipe(self, recipe: int = RECIPE_ROTCUBE, seed: int = 42):
        check(load().imb_group_init_recipe(self._h, int(recipe), C.c_uint64(seed)))

    def set_sync(self, mode: str):
        """'events' (default) or 'flags' (device flag words, fused slabs)."""
        check(load().imb_group_set_sync(self._h, {"events": 0, "flags": 1}[mode]))

    def run(self, steps: int):
        per = (C.c_double * len(self.teams))()
        wall = C.c_double()
        check(load().imb_group_run(self._h, int(steps), per, C.byref(wall)))
        return list(per), wall.value

    def download(self, field="x") -> np.ndarray:
        return np.concatenate([t.download(field) for t in self.teams], axis=0)
