"""Independent physics helpers used to PIN the oracle (tests only).

Nothing here is shared with the oracle or with the CUDA path: the detector
rotation comes from scipy's rotation-vector routine, and the tangent depth is
solved as the quadratic of SURVEY.md §8(c) "Pins" (i), in a 2-D frame
perpendicular to the wire axis, in extended precision.  The wire edge
(leading/trailing) is chosen physically: the contact point of the tangent line
on the wire side that faces (leading) or trails (trailing) the scan direction.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial.transform import Rotation

LD = np.longdouble


def det_rotation(rotvec) -> np.ndarray:
    return Rotation.from_rotvec(np.asarray(rotvec, dtype=np.float64)).as_matrix()


def detector_xyz(g: dict, x: float, j: float) -> np.ndarray:
    """Lab position of detector point (column coordinate x, row j), pixel centre i at (i-(C-1)/2)*pitch."""
    xp = (x - (g["n_cols"] - 1) / 2.0) * g["pitch_col"]
    yp = (j - (g["n_rows"] - 1) / 2.0) * g["pitch_row"]
    return det_rotation(g["det_rot"]) @ (np.array([xp, yp, 0.0]) + np.asarray(g["det_trans"], dtype=np.float64))


def _frame(axis):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    t = np.array([1.0, 0.0, 0.0]) if abs(a[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    u = t - (t @ a) * a
    u /= np.linalg.norm(u)
    v = np.cross(a, u)
    return a, u, v


def tangent_roots(Q, W, axis, r, beam=(0, 0, 1), origin=(0, 0, 0)):
    """Both beam depths z whose line to Q is tangent to the wire cylinder.

    2-D in the plane perpendicular to the axis (wire centre at the origin):
    q = pixel, p(z) = p0 + z*kappa = beam point.  Tangency: (q x p)^2 = r^2 |p - q|^2,
    a quadratic in z.  Returns (roots sorted ascending, contact points [2,2], frame).
    """
    a, u, v = _frame(axis)
    Q, W, O, k = (np.asarray(x, dtype=np.float64) for x in (Q, W, origin, beam))
    k = k / np.linalg.norm(k)
    q = np.array([LD((Q - W) @ u), LD((Q - W) @ v)])
    p0 = np.array([LD((O - W) @ u), LD((O - W) @ v)])
    kap = np.array([LD(k @ u), LD(k @ v)])
    cross = lambda s, t: s[0] * t[1] - s[1] * t[0]
    alpha, beta = cross(q, p0), cross(q, kap)
    dl = p0 - q
    r = LD(r)
    A = beta * beta - r * r * (kap @ kap)
    B = LD(2) * (alpha * beta - r * r * (dl @ kap))
    Cc = alpha * alpha - r * r * (dl @ dl)
    disc = B * B - LD(4) * A * Cc
    sq = np.sqrt(disc)
    # numerically stable pair
    qq = -(B + np.copysign(sq, B)) / LD(2)
    z1, z2 = qq / A, Cc / qq
    roots = sorted([z1, z2])
    contacts = []
    for z in roots:
        p = p0 + z * kap
        dvec = p - q
        uh = dvec / np.sqrt(dvec @ dvec)
        T = q + (-(q @ uh)) * uh  # foot of perpendicular from the wire centre
        contacts.append(T)
    return [float(z) for z in roots], np.array(contacts, dtype=np.float64), (a, u, v)


def edge_depth(Q, W, axis, r, scan_dir, edge="leading", beam=(0, 0, 1), origin=(0, 0, 0)) -> float:
    """Tangent depth for the wire edge facing (leading) / away from (trailing) the scan direction."""
    roots, contacts, (a, u, v) = tangent_roots(Q, W, axis, r, beam, origin)
    d = np.asarray(scan_dir, dtype=np.float64)
    d2 = np.array([d @ u, d @ v])
    side = contacts @ d2
    want = 1.0 if edge == "leading" else -1.0
    idx = int(np.argmax(want * side))
    return roots[idx]


def trapezoid_pdf(z, corners):
    """Unit-height trapezoid through sorted corners (0,1,1,0), vectorised."""
    z1, z2, z3, z4 = corners
    z = np.asarray(z, dtype=np.float64)
    up = np.where(z2 > z1, (z - z1) / np.where(z2 > z1, z2 - z1, 1.0), 1.0)
    dn = np.where(z4 > z3, (z4 - z) / np.where(z4 > z3, z4 - z3, 1.0), 1.0)
    h = np.minimum(np.minimum(up, dn), 1.0)
    return np.where((z < z1) | (z > z4), 0.0, np.maximum(h, 0.0))


def edge_depth_vec(Q, W, axis, r, scan_dir, edge="leading", beam=(0, 0, 1), origin=(0, 0, 0)):
    """Vectorised fp64 version of edge_depth: Q [n,3], W [n,3] -> depth [n]."""
    a, u, v = _frame(axis)
    Q = np.atleast_2d(np.asarray(Q, dtype=np.float64))
    W = np.atleast_2d(np.asarray(W, dtype=np.float64))
    O = np.asarray(origin, dtype=np.float64)
    k = np.asarray(beam, dtype=np.float64)
    k = k / np.linalg.norm(k)
    qx, qy = (Q - W) @ u, (Q - W) @ v
    px, py = (O - W) @ u, (O - W) @ v
    kx, ky = k @ u, k @ v
    alpha = qx * py - qy * px
    beta = qx * ky - qy * kx
    dx, dy = px - qx, py - qy
    A = beta * beta - r * r * (kx * kx + ky * ky)
    B = 2.0 * (alpha * beta - r * r * (dx * kx + dy * ky))
    Cc = alpha * alpha - r * r * (dx * dx + dy * dy)
    sq = np.sqrt(B * B - 4.0 * A * Cc)
    qq = -(B + np.copysign(sq, B)) / 2.0
    roots = np.stack([qq / A, Cc / qq], axis=1)
    d = np.asarray(scan_dir, dtype=np.float64)
    d2 = np.array([d @ u, d @ v])
    want = 1.0 if edge == "leading" else -1.0
    best = np.full(Q.shape[0], -np.inf)
    out = np.empty(Q.shape[0])
    for c in range(2):
        z = roots[:, c]
        ex, ey = px + z * kx - qx, py + z * ky - qy
        nrm = np.sqrt(ex * ex + ey * ey)
        ux, uy = ex / nrm, ey / nrm
        tq = -(qx * ux + qy * uy)
        tx, ty = qx + tq * ux, qy + tq * uy
        side = want * (tx * d2[0] + ty * d2[1])
        take = side > best
        out = np.where(take, z, out)
        best = np.where(take, side, best)
    return out


def occluded(P, Q, W, axis, r):
    """True where the segment P->Q passes within r of the wire axis line (W, axis). Vectorised.

    Independent forward (occlusion) model for round-trip tests: uses only the
    line-to-line distance, never a tangent construction.
    """
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    v = Q - P
    n = np.cross(a, v)
    nn = np.linalg.norm(n, axis=-1)
    dist = np.abs(np.sum((P - W) * n, axis=-1)) / nn
    # closest point parameter along the segment (must be inside it)
    w0 = P - W
    b = np.sum(a * v, axis=-1)
    c = np.sum(v * v, axis=-1)
    d = np.sum(a * w0, axis=-1)
    e = np.sum(v * w0, axis=-1)
    den = c - b * b
    lam = (b * d - e) / den
    return (dist < r) & (lam > 0.0) & (lam < 1.0)
