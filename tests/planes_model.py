"""numpy model of the direction-plane lattice step and its y-slab sharding —
test infrastructure mirroring csrc/lattice.cu + csrc/comm.cu on the CPU, so
the multi-GPU decomposition (which rows move where each step) can be checked
with the gloo backend on a machine without GPUs.

Arithmetic is numpy's, in the kernel's order, so results are bitwise equal to
the reference CSR step (asserted in tests/test_distributed_cpu.py).
"""

from __future__ import annotations

import numpy as np

D, L, R, U = 0, 1, 2, 3


def slot_dirs(nx: int, ny: int, gys) -> np.ndarray:
    """(len(gys), nx, 4) direction held by each reference slot."""
    gys = np.asarray(gys)
    x = np.arange(nx)
    xe = (x == 0) | (x == nx - 1)
    h0 = np.where(xe, R, L)
    h1 = np.where(xe, L, R)
    out = np.empty((gys.shape[0], nx, 4), dtype=np.int64)
    for i, gy in enumerate(gys):
        if gy == 0:
            out[i] = np.stack([h0, h1, np.full(nx, U), np.full(nx, D)], axis=1)
        elif gy == ny - 1:
            out[i] = np.stack([np.full(nx, U), np.full(nx, D), h0, h1], axis=1)
        else:
            out[i] = np.stack([np.full(nx, D), h0, h1, np.full(nx, U)], axis=1)
    return out


def arcs_to_planes(nx, ny, arcs, y0=0, rows=None, extra=0):
    rows = ny if rows is None else rows
    a = np.asarray(arcs).reshape(rows, nx, 4)
    d = slot_dirs(nx, ny, [(y0 + r) % ny for r in range(rows)])
    planes = np.zeros((4, rows + 2 * extra, nx), dtype=np.complex128)
    r_idx, x_idx = np.meshgrid(np.arange(rows), np.arange(nx), indexing="ij")
    for s in range(4):
        planes[d[:, :, s], r_idx + extra, x_idx] = a[:, :, s]
    return planes


def planes_to_arcs(nx, ny, planes, y0=0, rows=None, extra=0):
    rows = ny if rows is None else rows
    d = slot_dirs(nx, ny, [(y0 + r) % ny for r in range(rows)])
    r_idx, x_idx = np.meshgrid(np.arange(rows), np.arange(nx), indexing="ij")
    out = np.empty((rows, nx, 4), dtype=np.complex128)
    for s in range(4):
        out[:, :, s] = planes[d[:, :, s], r_idx + extra, x_idx]
    return out.reshape(-1)


def _outputs(nx, ny, vals, gys, marked_mask):
    """vals (4, rows, nx) -> O (4, rows, nx) indexed by direction e."""
    d = slot_dirs(nx, ny, gys)                       # (rows, nx, 4)
    s = np.stack([np.take_along_axis(vals.transpose(1, 2, 0), d[:, :, i:i + 1], axis=2)[:, :, 0]
                  for i in range(4)])               # s_i in slot order
    q = [np.multiply(0.5 + 0j, s[i]) for i in range(4)]
    n = [np.multiply(-0.5 + 0j, s[i]) for i in range(4)]
    t12 = q[1] + q[2]
    O = [n[0] + (t12 + q[3]), q[0] + ((n[1] + q[2]) + q[3]), q[0] + ((q[1] + n[2]) + q[3]),
         q[0] + (t12 + n[3])]
    out = np.empty_like(vals)
    for i in range(4):
        for e in range(4):
            sel = d[:, :, i] == e
            out[e][sel] = O[i][sel]
    if marked_mask is not None and marked_mask.any():
        neg = np.multiply(-1.0 + 0j, vals)
        out[:, marked_mask] = neg[:, marked_mask]
    return out


def step_slab(nx, ny, y0, rows, planes, shift="flipflop", marked=()):
    """One step of a slab (planes with one extra row each side); returns new
    planes whose extra rows hold the values pushed to the neighbours."""
    gys = [(y0 + r) % ny for r in range(rows)]
    vals = planes[:, 1:rows + 1, :]
    mask = None
    if marked:
        gv = (np.asarray(gys)[:, None] * nx + np.arange(nx)[None, :])
        mask = np.isin(gv, np.asarray(sorted(marked)))
    O = _outputs(nx, ny, vals, gys, mask)
    out = np.zeros_like(planes)
    sl = slice(1, rows + 1)
    if shift == "flipflop":
        out[U, 0:rows, :] = O[D]                      # below <- O_D (plane U)
        out[R, sl, :] = np.roll(O[L], -1, axis=1)     # left  <- O_L (plane R)
        out[L, sl, :] = np.roll(O[R], 1, axis=1)      # right <- O_R (plane L)
        out[D, 2:rows + 2, :] = O[U]                  # above <- O_U (plane D)
    else:
        out[D, 0:rows, :] = O[D]
        out[L, sl, :] = np.roll(O[L], -1, axis=1)
        out[R, sl, :] = np.roll(O[R], 1, axis=1)
        out[U, 2:rows + 2, :] = O[U]
    return out


def edge_planes(shift):
    """(plane sent down, plane sent up) — comm.cu's pd / pu."""
    return (U, D) if shift == "flipflop" else (D, U)


def exchange_local(slabs, shift):
    """Apply the per-step exchange to a list of slab planes (one process)."""
    pd, pu = edge_planes(shift)
    w = len(slabs)
    sends = [(s[pd, 0, :].copy(), s[pu, -1, :].copy()) for s in slabs]
    for i, s in enumerate(slabs):
        below, above = (i - 1) % w, (i + 1) % w
        rows = s.shape[1] - 2
        s[pd, rows, :] = sends[above][0]   # above's downward row -> my last owned row
        s[pu, 1, :] = sends[below][1]      # below's upward row -> my first owned row
    return slabs


def run_full(nx, ny, arcs, steps, shift="flipflop", marked=()):
    planes = arcs_to_planes(nx, ny, arcs, extra=1)
    for _ in range(steps):
        planes = step_slab(nx, ny, 0, ny, planes, shift, marked)
        exchange_local([planes], shift)
    return planes_to_arcs(nx, ny, planes, extra=1)


# ---- fused (ghost-row) slabs: csrc/comm.cu qwb_slab_run_fused ------------------

def ghost_window(nx, ny, arcs_owned, y0, rows, G):
    """Planes (4, rows + 2G, nx) of a slab with G ghost state rows each side
    (ghosts zero until the first exchange)."""
    w = np.zeros((4, rows + 2 * G, nx), dtype=np.complex128)
    w[:, G:G + rows, :] = arcs_to_planes(nx, ny, arcs_owned, y0, rows)
    return w


def ghost_steps(nx, ny, y0, rows, G, window, steps, shift="flipflop", marked=()):
    """`steps` (<= G) steps on the window with open y boundaries: after them
    the owned rows are exact (each step spoils one more window row per side)."""
    for _ in range(steps):
        padded = np.zeros((4, rows + 2 * G + 2, nx), dtype=np.complex128)
        padded[:, 1:-1, :] = window
        out = step_slab(nx, ny, y0 - G, rows + 2 * G, padded, shift, marked)
        window = out[:, 1:-1, :]
    return window


def ghost_sends(window, rows, G, g):
    """(rows for the rank below, rows for the rank above): the first / last g
    owned rows of every plane."""
    return window[:, G:G + g, :].copy(), window[:, G + rows - g:G + rows, :].copy()


def ghost_receive(window, rows, G, g, from_above, from_below):
    window[:, G + rows:G + rows + g, :] = from_above     # top ghost rows
    window[:, G - g:G, :] = from_below                   # bottom ghost rows
    return window
