// Exact triangle-mesh backend: the reference's OracleField / BruteForceField
// (field.py:144-215) over mesh.intersect_rays (mesh.py:264-279) and the numba
// kernels _ray_tri / _slab_enter / bvh_intersect (_kernels.py:43-204).
//
// Layout in HBM (built once on the host, mesh.py:94-166 median split):
//   nodes  64 B each: box lo/hi (f64), left, right, first triangle, count
//   tris   80 B each: the three vertices (f64) in leaf order + the face id
// One thread per ray walks the tree with a 64-entry stack in registers /
// local memory, near child first.  Every floating-point operation is an
// explicit round-to-nearest f64 op in the reference's order (no FMA
// contraction), and ties on t go to the lower face index, so the hit (face,
// t, u, v) is the reference's linear scan result bit for bit; the tree only
// decides which triangles are skipped.
#pragma once
#include "ddf_common.cuh"
#include "wavefront.cuh"

namespace ddf {
namespace mesh {

constexpr double DET_EPS = 1e-9;   // _kernels.py:16 Moller-Trumbore determinant cutoff
constexpr int STACK = 64;

struct Node {
  double lo[3], hi[3];
  int left, right, start, count;   // left < 0: leaf [start, start + count)
};
static_assert(sizeof(Node) == 64, "node layout");

struct Tri {
  double a[3], b[3], c[3];
  int face, pad;
};
static_assert(sizeof(Tri) == 80, "triangle layout");

struct MeshDev {
  const Node* nodes;
  const Tri* tris;
  const int* tri_of_face;   // face id -> position in tris
  int n_faces;
};

// _kernels.py:43-77
__device__ __forceinline__ double ray_tri(d3 o, d3 d, const Tri& T, double& u_out, double& v_out) {
  const double ax = T.a[0], ay = T.a[1], az = T.a[2];
  const double e1x = dsub(T.b[0], ax), e1y = dsub(T.b[1], ay), e1z = dsub(T.b[2], az);
  const double e2x = dsub(T.c[0], ax), e2y = dsub(T.c[1], ay), e2z = dsub(T.c[2], az);
  const double hx = dsub(dmul(d.y, e2z), dmul(d.z, e2y));
  const double hy = dsub(dmul(d.z, e2x), dmul(d.x, e2z));
  const double hz = dsub(dmul(d.x, e2y), dmul(d.y, e2x));
  const double det = dadd(dadd(dmul(e1x, hx), dmul(e1y, hy)), dmul(e1z, hz));
  if (-DET_EPS < det && det < DET_EPS) return INFINITY;
  const double f = ddiv(1.0, det);
  const double sx = dsub(o.x, ax), sy = dsub(o.y, ay), sz = dsub(o.z, az);
  const double u = dmul(f, dadd(dadd(dmul(sx, hx), dmul(sy, hy)), dmul(sz, hz)));
  if (u < 0.0 || u > 1.0) return INFINITY;
  const double qx = dsub(dmul(sy, e1z), dmul(sz, e1y));
  const double qy = dsub(dmul(sz, e1x), dmul(sx, e1z));
  const double qz = dsub(dmul(sx, e1y), dmul(sy, e1x));
  const double v = dmul(f, dadd(dadd(dmul(d.x, qx), dmul(d.y, qy)), dmul(d.z, qz)));
  if (v < 0.0 || dadd(u, v) > 1.0) return INFINITY;
  u_out = u;
  v_out = v;
  return dmul(f, dadd(dadd(dmul(e2x, qx), dmul(e2y, qy)), dmul(e2z, qz)));
}

// _kernels.py:80-127: entry t of the ray over [t0, t1] in the box, +inf on a miss
__device__ __forceinline__ double slab_enter(d3 o, d3 d, const double* lo, const double* hi, double t0, double t1) {
  double tmin = t0, tmax = t1;
  const double oc[3] = {o.x, o.y, o.z}, dc[3] = {d.x, d.y, d.z};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (dc[k] != 0.0) {
      const double inv = ddiv(1.0, dc[k]);
      double a = dmul(dsub(lo[k], oc[k]), inv);
      double b = dmul(dsub(hi[k], oc[k]), inv);
      if (a > b) { const double x = a; a = b; b = x; }
      if (a > tmin) tmin = a;
      if (b < tmax) tmax = b;
    } else if (oc[k] < lo[k] || oc[k] > hi[k]) {
      return INFINITY;
    }
  }
  if (tmin > tmax) return INFINITY;
  return tmin;
}

__device__ __forceinline__ void load_node(const Node* nodes, int i, double lo[3], double hi[3], int4& links) {
  const double2* p = reinterpret_cast<const double2*>(nodes + i);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
  lo[0] = a.x; lo[1] = a.y; lo[2] = b.x;
  hi[0] = b.y; hi[1] = c.x; hi[2] = c.y;
  links = __ldg(reinterpret_cast<const int4*>(nodes + i) + 3);
}

// _kernels.py:150-204 bvh_intersect: nearest hit with t in [t_min, t_max];
// face = -1 on a miss (t = inf, u = v = 0)
__device__ __forceinline__ void intersect(const MeshDev& M, d3 o, d3 d, double t_min, double t_max, int& bf,
                                          double& bt, double& bu, double& bv) {
  bf = -1;
  bt = INFINITY;
  bu = 0.0;
  bv = 0.0;
  int stack[STACK];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const int node = stack[--sp];
    const double limit = bt < t_max ? bt : t_max;
    double lo[3], hi[3];
    int4 ln;
    load_node(M.nodes, node, lo, hi, ln);
    if (slab_enter(o, d, lo, hi, t_min, limit) == INFINITY) continue;
    if (ln.x < 0) {
      for (int k = ln.z; k < ln.z + ln.w; ++k) {
        const Tri& T = M.tris[k];
        double u = 0.0, v = 0.0;
        const double t = ray_tri(o, d, T, u, v);
        if (t_min <= t && t <= t_max) {
          const int face = T.face;
          if (t < bt || (t == bt && face < bf)) {
            bf = face;
            bt = t;
            bu = u;
            bv = v;
          }
        }
      }
    } else {
      double llo[3], lhi[3], rlo[3], rhi[3];
      int4 dummy;
      load_node(M.nodes, ln.x, llo, lhi, dummy);
      load_node(M.nodes, ln.y, rlo, rhi, dummy);
      const double el = slab_enter(o, d, llo, lhi, t_min, limit);
      const double er = slab_enter(o, d, rlo, rhi, t_min, limit);
      // near child popped first (_kernels.py:187-203)
      if (el <= er) {
        if (er != INFINITY && sp < STACK) stack[sp++] = ln.y;
        if (el != INFINITY && sp < STACK) stack[sp++] = ln.x;
      } else {
        if (el != INFINITY && sp < STACK) stack[sp++] = ln.x;
        if (er != INFINITY && sp < STACK) stack[sp++] = ln.y;
      }
    }
  }
}

// mesh.intersect_rays (mesh.py:264-279)
__global__ void intersect_kernel(const MeshDev M, const double* o, const double* d, int n, double t_min,
                                 double t_max, int64_t* face, double* t, double* u, double* v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int f;
  double tt, uu, vv;
  intersect(M, ld3(o, i), ld3(d, i), t_min, t_max, f, tt, uu, vv);
  if (face) face[i] = f;
  if (t) t[i] = tt;
  if (u) u[i] = uu;
  if (v) v[i] = vv;
}

// _MeshField.query_batch / trace_batch (field.py:161-168): t (inf on miss), hit = face >= 0
__global__ void query_kernel(const MeshDev M, const double* o, const double* d, int n, double* t, uint8_t* hit,
                             double* pred, int* obj) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int f;
  double tt, uu, vv;
  intersect(M, ld3(o, i), ld3(d, i), 0.0, INFINITY, f, tt, uu, vv);
  t[i] = tt;
  hit[i] = f >= 0;
  if (pred) pred[i] = tt;
  if (obj) obj[i] = f;
}

// unnormalised geometric normal of a face: np.cross(v1 - v0, v2 - v0) (field.py:182)
__device__ __forceinline__ d3 face_cross(const MeshDev& M, int face) {
  const Tri& T = M.tris[M.tri_of_face[face]];
  const double e1x = dsub(T.b[0], T.a[0]), e1y = dsub(T.b[1], T.a[1]), e1z = dsub(T.b[2], T.a[2]);
  const double e2x = dsub(T.c[0], T.a[0]), e2y = dsub(T.c[1], T.a[1]), e2z = dsub(T.c[2], T.a[2]);
  return mk3(dsub(dmul(e1y, e2z), dmul(e1z, e2y)), dsub(dmul(e1z, e2x), dmul(e1x, e2z)),
             dsub(dmul(e1x, e2y), dmul(e1y, e2x)));
}

// _MeshField.normal_batch (field.py:172-189): re-intersect, face normal, n . d < 0
__global__ void normal_kernel(const MeshDev M, const double* o, const double* d, int n, double* nrm,
                              uint8_t* valid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const d3 di = ld3(d, i);
  int f;
  double tt, uu, vv;
  intersect(M, ld3(o, i), di, 0.0, INFINITY, f, tt, uu, vv);
  d3 r = mk3(0.0, 0.0, 0.0);
  if (f >= 0) {
    const d3 c = face_cross(M, f);
    const double nr = norm3(c);
    r = mk3(ddiv(c.x, nr), ddiv(c.y, nr), ddiv(c.z, nr));
    if (dot3(r, di) > 0.0) r = mk3(-r.x, -r.y, -r.z);
  }
  st3(nrm, i, r);
  valid[i] = f >= 0;
}

// render_path's trace_batch over path slots (all P, or the alive list):
// t, hit and the hit face (kept in S.obj for the normal stage)
__global__ void trace_paths_kernel(const MeshDev M, const PathState S, const int* list, const int* count, int P) {
  const int n = list ? *count : P;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int p = list ? list[k] : k;
    if (!S.march[p]) continue;
    int f;
    double tt, uu, vv;
    intersect(M, ld3(S.o, p), ld3(S.d, p), 0.0, INFINITY, f, tt, uu, vv);
    S.t[p] = tt;
    S.hit[p] = f >= 0;
    S.obj[p] = f;
    S.march[p] = 0;
  }
}

// render_path's normal_batch for the alive list: the hit face's cross product
// goes where a neural field's spatial gradient goes (S.g3); bounce_kernel
// normalises and flips it exactly like field.py:183-187.  (A face with
// |cross| < 1e-12 has |det| < 1e-9 for every ray, so it is never hit and the
// neural validity test never fires on a mesh.)
__global__ void face_normal_kernel(const MeshDev M, const PathState S, const int* list, const int* count) {
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int p = list[k];
    st3(S.g3, p, face_cross(M, S.obj[p]));
  }
}

// ------------------------------------------------------------ closest point
// _kernels.py:363-424 _point_tri_dist_sq (Ericson's region tests), same
// operation order; squared distance from p to triangle T.
__device__ __forceinline__ double point_tri_dist_sq(d3 p, const Tri& T) {
  const double ax = T.a[0], ay = T.a[1], az = T.a[2];
  const double bx = T.b[0], by = T.b[1], bz = T.b[2];
  const double cx = T.c[0], cy = T.c[1], cz = T.c[2];
  auto dot = [](double x0, double y0, double z0, double x1, double y1, double z1) {
    return dadd(dadd(dmul(x0, x1), dmul(y0, y1)), dmul(z0, z1));
  };
  const double abx = dsub(bx, ax), aby = dsub(by, ay), abz = dsub(bz, az);
  const double acx = dsub(cx, ax), acy = dsub(cy, ay), acz = dsub(cz, az);
  const double apx = dsub(p.x, ax), apy = dsub(p.y, ay), apz = dsub(p.z, az);
  const double d1 = dot(abx, aby, abz, apx, apy, apz);
  const double d2 = dot(acx, acy, acz, apx, apy, apz);
  if (d1 <= 0.0 && d2 <= 0.0) return dot(apx, apy, apz, apx, apy, apz);
  const double bpx = dsub(p.x, bx), bpy = dsub(p.y, by), bpz = dsub(p.z, bz);
  const double d3 = dot(abx, aby, abz, bpx, bpy, bpz);
  const double d4 = dot(acx, acy, acz, bpx, bpy, bpz);
  if (d3 >= 0.0 && d4 <= d3) return dot(bpx, bpy, bpz, bpx, bpy, bpz);
  const double vc = dsub(dmul(d1, d4), dmul(d3, d2));
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    const double den = dsub(d1, d3);
    const double w = den != 0.0 ? ddiv(d1, den) : 0.0;
    const double ex = dsub(apx, dmul(w, abx)), ey = dsub(apy, dmul(w, aby)), ez = dsub(apz, dmul(w, abz));
    return dot(ex, ey, ez, ex, ey, ez);
  }
  const double cpx = dsub(p.x, cx), cpy = dsub(p.y, cy), cpz = dsub(p.z, cz);
  const double d5 = dot(abx, aby, abz, cpx, cpy, cpz);
  const double d6 = dot(acx, acy, acz, cpx, cpy, cpz);
  if (d6 >= 0.0 && d5 <= d6) return dot(cpx, cpy, cpz, cpx, cpy, cpz);
  const double vb = dsub(dmul(d5, d2), dmul(d1, d6));
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    const double den = dsub(d2, d6);
    const double w = den != 0.0 ? ddiv(d2, den) : 0.0;
    const double ex = dsub(apx, dmul(w, acx)), ey = dsub(apy, dmul(w, acy)), ez = dsub(apz, dmul(w, acz));
    return dot(ex, ey, ez, ex, ey, ez);
  }
  const double va = dsub(dmul(d3, d6), dmul(d5, d4));
  const double e1 = dsub(d4, d3), e2 = dsub(d5, d6);
  if (va <= 0.0 && e1 >= 0.0 && e2 >= 0.0) {
    const double den = dadd(e1, e2);
    const double w = den != 0.0 ? ddiv(e1, den) : 0.0;
    const double ex = dsub(bpx, dmul(w, dsub(cx, bx)));
    const double ey = dsub(bpy, dmul(w, dsub(cy, by)));
    const double ez = dsub(bpz, dmul(w, dsub(cz, bz)));
    return dot(ex, ey, ez, ex, ey, ez);
  }
  const double denom = dadd(dadd(va, vb), vc);
  if (denom == 0.0) return dot(apx, apy, apz, apx, apy, apz);
  const double v = ddiv(vb, denom), w = ddiv(vc, denom);
  const double ex = dsub(dsub(apx, dmul(v, abx)), dmul(w, acx));
  const double ey = dsub(dsub(apy, dmul(v, aby)), dmul(w, acy));
  const double ez = dsub(dsub(apz, dmul(v, abz)), dmul(w, acz));
  return dot(ex, ey, ez, ex, ey, ez);
}

// _kernels.py:427-448
__device__ __forceinline__ double box_dist_sq(d3 p, const double* lo, const double* hi) {
  double d = 0.0;
  const double pc[3] = {p.x, p.y, p.z};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (pc[k] < lo[k]) {
      const double e = dsub(lo[k], pc[k]);
      d = dadd(d, dmul(e, e));
    } else if (pc[k] > hi[k]) {
      const double e = dsub(pc[k], hi[k]);
      d = dadd(d, dmul(e, e));
    }
  }
  return d;
}

// _kernels.py:451-500 closest_dist: exact point-to-surface distance; the
// minimum over triangles does not depend on the tree
__device__ __forceinline__ double closest(const MeshDev& M, d3 p) {
  double best = INFINITY;
  int stack[STACK];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const int node = stack[--sp];
    double lo[3], hi[3];
    int4 ln;
    load_node(M.nodes, node, lo, hi, ln);
    if (box_dist_sq(p, lo, hi) >= best) continue;
    if (ln.x < 0) {
      for (int k = ln.z; k < ln.z + ln.w; ++k) {
        const double dd = point_tri_dist_sq(p, M.tris[k]);
        if (dd < best) best = dd;
      }
    } else {
      double llo[3], lhi[3], rlo[3], rhi[3];
      int4 dummy;
      load_node(M.nodes, ln.x, llo, lhi, dummy);
      load_node(M.nodes, ln.y, rlo, rhi, dummy);
      const double dl = box_dist_sq(p, llo, lhi), dr = box_dist_sq(p, rlo, rhi);
      if (sp + 2 > STACK) continue;
      if (dl <= dr) { stack[sp++] = ln.y; stack[sp++] = ln.x; }
      else { stack[sp++] = ln.x; stack[sp++] = ln.y; }
    }
  }
  return sqrt(best);
}

__global__ void closest_kernel(const MeshDev M, const double* pts, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = closest(M, ld3(pts, i));
}

}  // namespace mesh
}  // namespace ddf
