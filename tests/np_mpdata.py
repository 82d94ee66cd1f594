"""Vectorised numpy restatement of the pinned MPDATA scheme.

Test-only second restatement, written independently of oracle/mpdata_oracle.c
with np.roll for the periodic shifts; it cross-checks the C oracle's stencil
indexing. Arrays are (n, m, l); face arrays use the staggered convention
u[i,j,k] at (i-1/2, j, k).
"""
import numpy as np

EPS = 1e-15


def sh(a, d, axis):
    """a shifted so that result[i] = a[i + d] along axis (periodic)."""
    return np.roll(a, -d, axis=axis)


def flux(a, b, c):
    return np.maximum(c, 0) * a + np.minimum(c, 0) * b


def update(x, U, V, W, h):
    fxl = flux(sh(x, -1, 0), x, U)
    fxr = sh(fxl, 1, 0)
    fyl = flux(sh(x, -1, 1), x, V)
    fyr = sh(fyl, 1, 1)
    fzl = flux(sh(x, -1, 2), x, W)
    fzr = sh(fzl, 1, 2)
    return x - (((fxr - fxl) + (fyr - fyl)) + (fzr - fzl)) / h


def ratio(a, b, eps):
    return (a - b) / ((a + b) + eps)


def pseudo(x, U, V, W, h, eps=EPS):
    a = np.abs(x)
    vel = [U, V, W]
    out = []
    for ax in range(3):
        t1, t2 = [q for q in range(3) if q != ax]
        Un = vel[ax]
        hb = 0.5 * (sh(h, -1, ax) + h)
        A = ratio(a, sh(a, -1, ax), eps)
        terms = []
        for t in (t1, t2):
            aL = sh(a, -1, ax)
            sp = sh(aL, 1, t) + sh(a, 1, t)
            sm = sh(aL, -1, t) + sh(a, -1, t)
            B = ratio(sp, sm, eps)
            Vt = vel[t]
            S = (sh(Vt, -1, ax) + Vt) + (sh(sh(Vt, -1, ax), 1, t) + sh(Vt, 1, t))
            terms.append((S, B))
        (S1, B1), (S2, B2) = terms
        t1v = (np.abs(Un) - (Un * Un) / hb) * A
        cr = S1 * B1 + S2 * B2
        out.append(t1v - ((0.125 * Un) * cr) / hb)
    return out


def ext7(x, fn):
    r = x
    for ax in range(3):
        for d in (-1, 1):
            r = fn(r, sh(x, d, ax))
    return r


def step(x, u, v, w, h, iord=2, nonos=True, eps=EPS):
    xn = x
    cur = update(x, u, v, w, h)
    U, V, W = u, v, w
    mx = mn = None
    for k in range(2, iord + 1):
        ut, vt, wt = pseudo(cur, U, V, W, h, eps)
        if nonos:
            if k == 2:
                mx = np.maximum(ext7(cur, np.maximum), ext7(xn, np.maximum))
                mn = np.minimum(ext7(cur, np.minimum), ext7(xn, np.minimum))
            else:
                mx = np.maximum(ext7(cur, np.maximum), mx)
                mn = np.minimum(ext7(cur, np.minimum), mn)
            fl = [flux(sh(cur, -1, a), cur, vv) for a, vv in enumerate((ut, vt, wt))]
            fr = [sh(f, 1, a) for a, f in enumerate(fl)]
            pos = lambda q: np.maximum(q, 0)  # noqa: E731
            neg = lambda q: np.minimum(q, 0)  # noqa: E731
            fin = ((pos(fl[0]) - neg(fr[0])) + (pos(fl[1]) - neg(fr[1]))) + (pos(fl[2]) - neg(fr[2]))
            fout = ((pos(fr[0]) - neg(fl[0])) + (pos(fr[1]) - neg(fl[1]))) + (pos(fr[2]) - neg(fl[2]))
            bu = ((mx - cur) * h) / (fin + eps)
            bd = ((cur - mn) * h) / (fout + eps)
            lim = []
            for a, vv in enumerate((ut, vt, wt)):
                cp = np.minimum(np.minimum(1.0, sh(bd, -1, a)), bu)
                cn = np.minimum(np.minimum(1.0, sh(bu, -1, a)), bd)
                lim.append(pos(vv) * cp + neg(vv) * cn)
            ut, vt, wt = lim
        cur = update(cur, ut, vt, wt, h)
        U, V, W = ut, vt, wt
    return cur
