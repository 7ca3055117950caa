"""TEST INFRASTRUCTURE ONLY - numpy restatement of the reference LETKF arm.

Follows ``/root/reference/proj/src/letkf.cpp`` line by line (per grid point,
in the reference's gather order) so the GPU LETKF (``csrc/letkf_kernels.cu``,
which uses a different but equivalent formulation: a periodic convolution of
per-cell outer products and a batched Jacobi eigensolver) can be checked
against it.  The reference itself needs Eigen, which is absent from this
image, so it cannot be built here: **parity unpinned** for the LETKF arm.
What pins it instead: the closed-form and property tests of the reference's
own ``proj/tests/test_letkf.cpp`` (restated in ``tests/test_letkf_oracle.py``
and ``tests/test_gpu_letkf.py``).

Only ``tests/`` may import this module.
"""
from __future__ import annotations

import math

import numpy as np


def gaspari_cohn(r: float) -> float:
    """proj/src/letkf.cpp:10-18 (5th-order piecewise rational, support [0, 2])."""
    if r < 0.0:
        raise ValueError("gaspari_cohn: r >= 0")
    if r >= 2.0:
        return 0.0
    r2 = r * r
    r3 = r2 * r
    r4 = r3 * r
    r5 = r4 * r
    if r <= 1.0:
        return 1.0 - 5.0 / 3.0 * r2 + 5.0 / 8.0 * r3 + 0.5 * r4 - 0.25 * r5
    return (4.0 - 5.0 * r + 5.0 / 3.0 * r2 + 5.0 / 8.0 * r3 - 0.5 * r4 + r5 / 12.0
            - 2.0 / (3.0 * r))


def etkf_local_analysis(yb_pert, y, yb_mean, r_inv, m):
    """proj/src/letkf.cpp:20-55 (Hunt et al. 2007): returns (wbar, W)."""
    p = yb_pert.shape[0]
    if p == 0:
        return np.zeros(m), np.eye(m)
    c = yb_pert.T * r_inv[None, :]                      # M x p
    a = c @ yb_pert
    a[np.diag_indices(m)] += float(m - 1)
    lam, v = np.linalg.eigh(a)
    if not np.all(np.isfinite(lam)) or np.any(lam <= 0.0):
        raise ArithmeticError("singular local analysis")
    pa = (v / lam[None, :]) @ v.T
    wbar = pa @ (c @ (y - yb_mean))
    w = math.sqrt(m - 1) * ((v / np.sqrt(lam)[None, :]) @ v.T)
    return wbar, w


def localization_offsets(nx, ny, cutoff):
    """The gather stencil of proj/src/letkf.cpp:101-121: (ox, oy, gc) in the
    reference's loop order."""
    reach = min(int(math.ceil(2.0 * cutoff)), nx // 2)
    lo_x, hi_x = ((-nx // 2 + 1, nx // 2) if 2 * reach >= nx else (-reach, reach))
    lo_y, hi_y = ((-ny // 2 + 1, ny // 2) if 2 * reach >= ny else (-reach, reach))
    out = []
    for oy in range(lo_y, hi_y + 1):
        for ox in range(lo_x, hi_x + 1):
            ax = min(abs(ox), nx - abs(ox))
            ay = min(abs(oy), ny - abs(oy))
            r = math.hypot(ax, ay) / cutoff
            if r >= 2.0:
                continue
            out.append((ox, oy, gaspari_cohn(r)))
    return out


def grid_locations(nx, ny, obs_idx, d):
    """operator_locations, proj/src/observation.cpp:43-60."""
    q = np.arange(d) if obs_idx is None else np.asarray(obs_idx)
    h = q % (nx * ny)
    return np.stack([h % nx, h // nx], axis=1).astype(np.float64)


def rtps_inflate(analysis, background, alpha):
    """proj/src/letkf.cpp:177-207."""
    if alpha == 0.0:
        return analysis.copy()
    m = analysis.shape[0]
    if m < 2:
        return analysis.copy()
    ma = analysis.mean(axis=0)
    mb = background.mean(axis=0)
    va = ((analysis - ma) ** 2).sum(axis=0)
    vb = ((background - mb) ** 2).sum(axis=0)
    sa = np.maximum(np.sqrt(va / (m - 1)), 1e-12)
    sb = np.sqrt(vb / (m - 1))
    scale = 1.0 + alpha * (sb - sa) / sa
    return ma + scale * (analysis - ma)


def letkf_analyze(x, y, r, obs_idx, nx, ny, cutoff_km=2000.0, domain_km=20000.0,
                  rtps_alpha=0.3, arctan=False, locations=None):
    """letkf_analyze, proj/src/letkf.cpp:57-175, for grid operators (identity
    when ``obs_idx`` is None, else index selection; ``arctan`` applies
    h(x) = atan(x) on top, the north-star extension).  ``x``: (M, d) with
    d = 2*nx*ny.  Returns the (M, d) analysis after RTPS."""
    x = np.asarray(x, np.float64)
    m, d = x.shape
    if nx != ny:
        raise ValueError("letkf_analyze: isotropic metric needs nx == ny")
    if d != 2 * nx * ny:
        raise ValueError("letkf_analyze: state/grid size mismatch")
    y = np.asarray(y, np.float64)
    r = np.broadcast_to(np.asarray(r, np.float64), y.shape)
    cutoff = cutoff_km / domain_km * nx
    # obs-space background (:82-91)
    hx = x if obs_idx is None else x[:, np.asarray(obs_idx)]
    if arctan:
        hx = np.arctan(hx)
    hxb = hx.T.copy()                                   # p_total x M
    hxb_mean = hxb.mean(axis=1)
    hxb -= hxb_mean[:, None]
    xb_mean = x.mean(axis=0)
    locs = grid_locations(nx, ny, obs_idx, d) if locations is None else locations
    # bucket observations by integer cell (:96-101)
    cell_obs = [[] for _ in range(nx * ny)]
    for k in range(y.size):
        cx = int(math.floor(locs[k, 0])) % nx
        cy = int(math.floor(locs[k, 1])) % ny
        cell_obs[cy * nx + cx].append(k)
    offsets = localization_offsets(nx, ny, cutoff)
    xa = x.copy()
    for pt in range(nx * ny):
        ix, iy = pt % nx, pt // nx
        local, local_gc = [], []
        for ox, oy, gc in offsets:
            cx = (ix + ox % nx + nx) % nx
            cy = (iy + oy % ny + ny) % ny
            for k in cell_obs[cy * nx + cx]:
                local.append(k)
                local_gc.append(gc)
        if not local:
            continue
        local = np.asarray(local)
        rinv = np.asarray(local_gc) / r[local]
        wbar, w = etkf_local_analysis(hxb[local], y[local], hxb_mean[local], rinv, m)
        for row in (iy * nx + ix, nx * ny + iy * nx + ix):
            mean = xb_mean[row]
            pert = x[:, row] - mean
            wx = pert @ wbar
            pw = w.T @ pert
            xa[:, row] = mean + wx + pw
    return rtps_inflate(xa, x, rtps_alpha)
