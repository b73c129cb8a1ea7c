// Signed distance to a closed indexed triangle mesh, for ks_tsdf_stamp_mesh.
//
// The reference has NO mesh implementation (SPEC.md:8 and :422 put triangle-mesh stamping out of scope;
// PAPER.md:293 says only "Cuboids and meshes are stamped directly into the geometry channel"), so the
// definition is this repo's own, modelled on stamp_primitive (sdf_world.hpp:394-444) with the analytic
// distance replaced by:
//   magnitude = distance to the closest point over all triangles (region walk of the closest-point-on-
//               triangle problem, Ericson, "Real-Time Collision Detection" 5.1.5); among triangles at exactly
//               the same squared distance the lowest index wins;
//   sign      = sign of (p - closest) . pseudonormal of the feature the closest point lies on (face normal /
//               sum of the adjacent face normals for an edge / angle-weighted sum for a vertex); +0 on the surface.
// Every fp64 expression is written in one fixed order (length-3 reductions as a0 + (a1 + a2), like the rest of
// the library) and the library is built with -fmad=false, so a CPU restatement in the same order reproduces the
// values bit for bit.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace ksb {

struct MeshView {
  int nt;
  const double* tri;  // nt x {a, b, c}
  const double* nrm;  // nt x 7 pseudonormals: face, vertex a, b, c, edge ab, bc, ca
  const double* bnd;  // nt x {centre xyz, radius}: a sphere that contains the triangle (culling only)
};

struct V3 {
  double x, y, z;
};
__host__ __device__ __forceinline__ V3 v3(double x, double y, double z) { return V3{x, y, z}; }
__host__ __device__ __forceinline__ V3 v3_sub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
__host__ __device__ __forceinline__ double v3_dot(V3 a, V3 b) { return sum3(a.x * b.x, a.y * b.y, a.z * b.z); }
__host__ __device__ __forceinline__ V3 v3_axpy(V3 a, double s, V3 d) { return v3(a.x + s * d.x, a.y + s * d.y, a.z + s * d.z); }
__host__ __device__ __forceinline__ V3 v3_cross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// closest point of triangle (a, b, c) to p; feature: 0 face, 1..3 vertex a/b/c, 4 edge ab, 5 edge bc, 6 edge ca
__host__ __device__ __forceinline__ V3 closest_on_triangle(V3 p, V3 a, V3 b, V3 c, int& feature) {
  const V3 ab = v3_sub(b, a), ac = v3_sub(c, a), ap = v3_sub(p, a);
  const double d1 = v3_dot(ab, ap), d2 = v3_dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return feature = 1, a;
  const V3 bp = v3_sub(p, b);
  const double d3 = v3_dot(ab, bp), d4 = v3_dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return feature = 2, b;
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return feature = 4, v3_axpy(a, d1 / (d1 - d3), ab);
  const V3 cp = v3_sub(p, c);
  const double d5 = v3_dot(ab, cp), d6 = v3_dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return feature = 3, c;
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return feature = 6, v3_axpy(a, d2 / (d2 - d6), ac);
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0)
    return feature = 5, v3_axpy(b, (d4 - d3) / ((d4 - d3) + (d5 - d6)), v3_sub(c, b));
  const double denom = 1.0 / (va + (vb + vc));
  feature = 0;
  return v3_axpy(v3_axpy(a, vb * denom, ab), vc * denom, ac);
}

// running minimum over triangles: squared distance, then triangle index
struct MeshHit {
  double d2;
  int tri, feature;
  V3 diff;
};
__device__ __forceinline__ void mesh_visit(const MeshView& M, int j, V3 p, MeshHit& best) {
  const double* T = M.tri + 9 * static_cast<size_t>(j);
  int feature;
  const V3 q = closest_on_triangle(p, v3(__ldg(T), __ldg(T + 1), __ldg(T + 2)), v3(__ldg(T + 3), __ldg(T + 4), __ldg(T + 5)),
                                   v3(__ldg(T + 6), __ldg(T + 7), __ldg(T + 8)), feature);
  const V3 diff = v3_sub(p, q);
  const double d2 = v3_dot(diff, diff);
  if (d2 < best.d2 || (d2 == best.d2 && j < best.tri)) best.d2 = d2, best.tri = j, best.feature = feature, best.diff = diff;
}
__device__ __forceinline__ double mesh_signed(const MeshView& M, const MeshHit& h) {
  const double* N = M.nrm + 21 * static_cast<size_t>(h.tri) + 3 * h.feature;
  const double dist = sqrt(h.d2);
  return v3_dot(h.diff, v3(__ldg(N), __ldg(N + 1), __ldg(N + 2))) < 0.0 ? -dist : dist;
}
// distance from q to the centre of triangle j's bounding sphere, and that sphere's radius
__device__ __forceinline__ double mesh_bound(const MeshView& M, int j, V3 q, double& radius) {
  const double2 b0 = __ldg(reinterpret_cast<const double2*>(M.bnd) + 2 * j), b1 = __ldg(reinterpret_cast<const double2*>(M.bnd) + 2 * j + 1);
  radius = b1.y;
  const V3 d = v3(q.x - b0.x, q.y - b0.y, q.z - b1.x);
  return sqrt(v3_dot(d, d));
}
// Culling is conservative by a wide margin next to fp64 rounding (bounds are compared with 1e-6 relative slack on
// top of geometric inequalities that hold exactly), so it never changes which triangle wins.
constexpr double kMeshSlack = 1.000001;

// ---- host: validation and the per-triangle tables -----------------------------------------------------------
struct MeshTables {
  std::vector<double> tri, nrm, bnd;
  double lo[3], hi[3];  // AABB of all vertices
};

inline V3 v3_unit(V3 a) {  // v / sqrt(v.v), true divisions
  const double z = v3_dot(a, a);
  if (z > 0.0) {
    const double n = std::sqrt(z);
    return v3(a.x / n, a.y / n, a.z / n);
  }
  return a;
}
inline double corner_angle(V3 e1, V3 e2) {
  double c = v3_dot(v3_unit(e1), v3_unit(e2));
  c = c < -1.0 ? -1.0 : (1.0 < c ? 1.0 : c);
  return std::acos(c);
}

// nullptr on success, else the message of the validation failure
inline const char* build_mesh_tables(const double* vertices, int nv, const int32_t* triangles, int nt, MeshTables& out) {
  if (!vertices || !triangles || nv <= 0 || nt <= 0) return "stamp: empty mesh";
  for (long i = 0; i < 3L * nv; ++i)
    if (!std::isfinite(vertices[i])) return "stamp: non-finite mesh";
  for (long i = 0; i < 3L * nt; ++i)
    if (triangles[i] < 0 || triangles[i] >= nv) return "stamp: mesh index out of range";
  out.tri.assign(9 * static_cast<size_t>(nt), 0.0);
  out.nrm.assign(21 * static_cast<size_t>(nt), 0.0);
  out.bnd.assign(4 * static_cast<size_t>(nt), 0.0);
  std::vector<double> vn(3 * static_cast<size_t>(nv), 0.0);
  struct EdgeRef {
    int32_t lo, hi;
    int tri, side;
  };
  std::vector<EdgeRef> edges(3 * static_cast<size_t>(nt));
  auto vert = [&](int i) { return v3(vertices[3 * i], vertices[3 * i + 1], vertices[3 * i + 2]); };
  for (int i = 0; i < nt; ++i) {
    const int32_t* I = triangles + 3 * static_cast<size_t>(i);
    const V3 p[3] = {vert(I[0]), vert(I[1]), vert(I[2])};
    for (int k = 0; k < 3; ++k) out.tri[9 * i + 3 * k] = p[k].x, out.tri[9 * i + 3 * k + 1] = p[k].y, out.tri[9 * i + 3 * k + 2] = p[k].z;
    const V3 n = v3_cross(v3_sub(p[1], p[0]), v3_sub(p[2], p[0]));
    if (!(v3_dot(n, n) > 0.0)) return "stamp: degenerate mesh triangle";
    const V3 nf = v3_unit(n);
    out.nrm[21 * i] = nf.x, out.nrm[21 * i + 1] = nf.y, out.nrm[21 * i + 2] = nf.z;
    const double w[3] = {corner_angle(v3_sub(p[1], p[0]), v3_sub(p[2], p[0])), corner_angle(v3_sub(p[0], p[1]), v3_sub(p[2], p[1])),
                         corner_angle(v3_sub(p[0], p[2]), v3_sub(p[1], p[2]))};
    for (int k = 0; k < 3; ++k) {  // angle-weighted vertex pseudonormals, accumulated in triangle order
      vn[3 * I[k]] += w[k] * nf.x, vn[3 * I[k] + 1] += w[k] * nf.y, vn[3 * I[k] + 2] += w[k] * nf.z;
      const int32_t a = I[k], b = I[(k + 1) % 3];
      edges[3 * static_cast<size_t>(i) + k] = EdgeRef{std::min(a, b), std::max(a, b), i, k};
    }
    // bounding sphere about the centroid (culling only; padded against rounding)
    const V3 m = v3((p[0].x + p[1].x + p[2].x) / 3.0, (p[0].y + p[1].y + p[2].y) / 3.0, (p[0].z + p[1].z + p[2].z) / 3.0);
    double r2 = 0.0;
    for (int k = 0; k < 3; ++k) r2 = std::max(r2, v3_dot(v3_sub(p[k], m), v3_sub(p[k], m)));
    out.bnd[4 * i] = m.x, out.bnd[4 * i + 1] = m.y, out.bnd[4 * i + 2] = m.z, out.bnd[4 * i + 3] = std::sqrt(r2) * kMeshSlack;
  }
  std::sort(edges.begin(), edges.end(), [](const EdgeRef& a, const EdgeRef& b) {
    if (a.lo != b.lo) return a.lo < b.lo;
    if (a.hi != b.hi) return a.hi < b.hi;
    return a.tri < b.tri;
  });
  for (size_t s = 0; s < edges.size();) {  // edge pseudonormal = sum of its faces' normals, in triangle order
    size_t e = s;
    double sum[3] = {0.0, 0.0, 0.0};
    for (; e < edges.size() && edges[e].lo == edges[s].lo && edges[e].hi == edges[s].hi; ++e)
      for (int ax = 0; ax < 3; ++ax) sum[ax] += out.nrm[21 * static_cast<size_t>(edges[e].tri) + ax];
    for (size_t k = s; k < e; ++k)
      for (int ax = 0; ax < 3; ++ax) out.nrm[21 * static_cast<size_t>(edges[k].tri) + 3 * (4 + edges[k].side) + ax] = sum[ax];
    s = e;
  }
  for (int i = 0; i < nt; ++i)
    for (int k = 0; k < 3; ++k)
      for (int ax = 0; ax < 3; ++ax) out.nrm[21 * static_cast<size_t>(i) + 3 * (1 + k) + ax] = vn[3 * static_cast<size_t>(triangles[3 * i + k]) + ax];
  for (int ax = 0; ax < 3; ++ax) out.lo[ax] = INFINITY, out.hi[ax] = -INFINITY;
  for (int i = 0; i < nv; ++i)
    for (int ax = 0; ax < 3; ++ax) {
      if (vertices[3 * i + ax] < out.lo[ax]) out.lo[ax] = vertices[3 * i + ax];
      if (out.hi[ax] < vertices[3 * i + ax]) out.hi[ax] = vertices[3 * i + ax];
    }
  return nullptr;
}

}  // namespace ksb
