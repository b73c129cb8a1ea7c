"""An INDEPENDENT signed distance to a closed triangle mesh, for checking csrc/mesh.cuh and oracle/ks_oracle.c's ko_mesh_sdf.

Deliberately a different algorithm on both halves (test infrastructure only; fp64 numpy, brute force):
  magnitude : per triangle, project the point onto the triangle's plane; if the projection's barycentric coordinates
              are all >= 0 the plane distance is the answer, otherwise the minimum over the three edge SEGMENTS
              (clamped parameter).  The product walks Ericson's seven Voronoi regions instead.
  sign      : the generalised winding number -- the sum of the signed solid angles of all triangles seen from the
              point (Van Oosterom & Strackee 1983), divided by 4 pi: +-1 inside a closed oriented mesh, 0 outside.
              The product takes the sign of (p - closest) . pseudonormal of the closest feature instead.
The two agree for every point that is not on the surface; the tests below skip points closer to it than 1e-9.
"""
import numpy as np


def _segment_d2(p, a, b):
    ab = b - a
    t = np.clip(((p - a) * ab).sum(-1) / (ab * ab).sum(-1), 0.0, 1.0)
    q = a + t[..., None] * ab
    return ((p - q) ** 2).sum(-1)


def unsigned_distance(vertices, triangles, points, chunk=2048):
    v = np.asarray(vertices, np.float64)
    tri = np.asarray(triangles, np.int64)
    a, b, c = v[tri[:, 0]][None], v[tri[:, 1]][None], v[tri[:, 2]][None]  # [1, T, 3]
    n = np.cross(b - a, c - a)
    nn = (n * n).sum(-1)
    out = np.empty(len(points))
    for s in range(0, len(points), chunk):
        p = np.asarray(points[s:s + chunk], np.float64)[:, None, :]  # [P, 1, 3]
        ap = p - a
        dist_plane = (ap * n).sum(-1)  # times |n|
        proj = p - (dist_plane / nn)[..., None] * n
        # barycentric coordinates of the projection through sub-triangle normals
        w_a = (np.cross(b - proj, c - proj) * n).sum(-1)
        w_b = (np.cross(c - proj, a - proj) * n).sum(-1)
        w_c = (np.cross(a - proj, b - proj) * n).sum(-1)
        inside = (w_a >= 0) & (w_b >= 0) & (w_c >= 0)
        d2_face = dist_plane ** 2 / nn
        d2_edges = np.minimum(np.minimum(_segment_d2(p, a, b), _segment_d2(p, b, c)), _segment_d2(p, c, a))
        d2 = np.where(inside, np.minimum(d2_face, d2_edges), d2_edges)
        out[s:s + chunk] = np.sqrt(d2.min(axis=1))
    return out


def winding_number(vertices, triangles, points, chunk=2048):
    v = np.asarray(vertices, np.float64)
    tri = np.asarray(triangles, np.int64)
    out = np.empty(len(points))
    for s in range(0, len(points), chunk):
        p = np.asarray(points[s:s + chunk], np.float64)[:, None, :]
        a, b, c = v[tri[:, 0]][None] - p, v[tri[:, 1]][None] - p, v[tri[:, 2]][None] - p
        la, lb, lc = np.linalg.norm(a, axis=-1), np.linalg.norm(b, axis=-1), np.linalg.norm(c, axis=-1)
        num = (a * np.cross(b, c)).sum(-1)
        den = la * lb * lc + (a * b).sum(-1) * lc + (b * c).sum(-1) * la + (c * a).sum(-1) * lb
        out[s:s + chunk] = (2.0 * np.arctan2(num, den)).sum(axis=1) / (4.0 * np.pi)
    return out


def signed_distance(vertices, triangles, points):
    """(signed distance, |winding number|): negative inside a closed, outward (counter-clockwise) oriented mesh."""
    d = unsigned_distance(vertices, triangles, points)
    w = winding_number(vertices, triangles, points)
    return np.where(np.abs(w) > 0.5, -d, d), np.abs(w)


# ---- non-convex closed test meshes (outward orientation) ------------------------------------------------------------
def torus(center, major, minor, nu=24, nv=12):
    """Ring torus around the z axis through `center`: genus 1, concave inner half."""
    center = np.asarray(center, np.float64)
    verts = []
    for i in range(nu):
        u = 2 * np.pi * i / nu
        for j in range(nv):
            w = 2 * np.pi * j / nv
            r = major + minor * np.cos(w)
            verts.append(center + np.array([r * np.cos(u), r * np.sin(u), minor * np.sin(w)]))
    tris = []
    for i in range(nu):
        for j in range(nv):
            p00, p10 = i * nv + j, ((i + 1) % nu) * nv + j
            p01, p11 = i * nv + (j + 1) % nv, ((i + 1) % nu) * nv + (j + 1) % nv
            tris += [[p00, p10, p11], [p00, p11, p01]]
    return np.array(verts), np.array(tris, np.int32)


def l_prism(origin, arm=0.3, thick=0.12, height=0.2):
    """L-shaped prism (a reflex edge along z): the polygon is extruded from z = 0 to `height`."""
    o = np.asarray(origin, np.float64)
    poly = np.array([[0, 0], [arm, 0], [arm, thick], [thick, thick], [thick, arm], [0, arm]], np.float64)  # counter-clockwise
    n = len(poly)
    verts = np.array([[x, y, 0.0] for x, y in poly] + [[x, y, height] for x, y in poly]) + o
    tris = []
    for i in range(n):  # side walls, outward
        j = (i + 1) % n
        tris += [[i, j, n + j], [i, n + j, n + i]]
    caps = [[0, 1, 2], [0, 2, 3], [0, 3, 4], [0, 4, 5]]  # fan from the reflex-free corner: all inside the L
    for a, b, c in caps:
        tris.append([a, c, b])              # bottom cap looks down
        tris.append([n + a, n + b, n + c])  # top cap looks up
    return verts, np.array(tris, np.int32)
