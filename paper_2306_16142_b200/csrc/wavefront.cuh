// Wavefront path tracer: render.render_path (render.py:198-247) as a sequence
// of stream-ordered kernels over a structure-of-arrays path state in HBM.
//
// A "wave" is a block of path slots p = (sample s, owned pixel q): s = s0 +
// p / n_own, pixel i = pix[q].  Every random draw is addressed by the GLOBAL
// pixel index i through PCG64 jump-ahead, so tiles, waves and rank count never
// change a draw:
//   jitter      draw k = (s(B+1) + 0)   * 2N + 2i + c      (render.py:213)
//   bounce b    draw k = (s(B+1) + 1+b) * 2N + 2i + c      (render.py:222)
//   RR (EXT.)   draw k = (s B + b) * N + i  of the separate RR stream
#pragma once
#include "ddf_common.cuh"
#include "field_kernels.cuh"

namespace ddf {

struct CamDev {
  double pos[3], fwd[3], right[3], up[3];
  double tan_half, aspect;
  int W, H;
};

struct PathState {
  double* o; double* d;            // (P,3)
  double* t_acc; double* t_exit; double* t;   // t = trace result (inf on miss)
  double* thr; double* rad;
  uint8_t* hit; uint8_t* march; uint8_t* alive;
  int* obj;
  double* u34;                     // (P,2) encoded angles of d (neural.py:36-37), set at ray creation
  double* g3;                      // (P,3) spatial input gradient from the gradient pass
  uint8_t* gdone;                  // 1: g3 already holds this segment's normal gradient (TraceGradOp)
  uint8_t* want;                   // 1: this segment's normal will be needed and may come from its first march step
};

struct WaveDev {
  int spp, bounces;
  double albedo, env;
  int rr_start;                 // -1: off
  int64_t n_pix;                // global film size W*H
  const int* pix;               // owned global pixel ids, ascending
  int n_own;
  int s0, ns;                   // samples of this wave
  const PcgStream* rng;         // render.py:209 stream
  const PcgStream* rr;          // EXTENSION stream
  int* err;                     // device error word (DevError bits)
  unsigned long long* degenerate;   // count of degenerate normals (render.py:133-136)
};

__device__ __forceinline__ void slot_sp(const WaveDev& w, int p, int& s, int& i) {
  s = w.s0 + p / w.n_own;
  i = w.pix[p % w.n_own];
}

// slab test + march initialisation for a new ray (field.py:265-269)
__device__ __forceinline__ void begin_trace(const FieldDev& F, const PathState& S, int p, d3 o, d3 d) {
  if (S.gdone) S.gdone[p] = 0;
  if (F.is_mesh) {   // mesh fields trace every ray exactly (field.py:161-168), no domain box
    S.march[p] = 1;
    S.t[p] = INFINITY;
    S.hit[p] = 0;
    S.obj[p] = -1;
    return;
  }
  double u3, u4;
  dir_u34(d, u3, u4);
  S.u34[2 * p] = u3;
  S.u34[2 * p + 1] = u4;
  double te, tx;
  ray_box(o, d, F.lo, F.hi, te, tx);
  const bool in = (te < tx) && (tx > 0.0);
  S.t_acc[p] = in ? fmax(te, 0.0) : 0.0;
  S.t_exit[p] = tx;
  S.march[p] = in;
  S.t[p] = INFINITY;
  S.hit[p] = 0;
  S.obj[p] = 0;
}

// primary rays: render.py:213-220 + pixel_rays render.py:54-75
#ifndef DDF_OPS_ONLY
__global__ void camera_kernel(const FieldDev F, const CamDev C, const WaveDev w, const PathState S, int P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int s, i;
  slot_sp(w, p, s, i);
  double ox, oy;
  pcg_pair(*w.rng, (uint64_t)(s * (w.bounces + 1)) * 2ull * (uint64_t)w.n_pix + 2ull * (uint64_t)i, ox, oy);
  const double px = (double)(i % C.W), py = (double)(i / C.W);
  const double sx = dmul(dmul(dsub(ddiv(dmul(2.0, dadd(px, ox)), (double)C.W), 1.0), C.tan_half), C.aspect);
  const double sy = dmul(dsub(1.0, ddiv(dmul(2.0, dadd(py, oy)), (double)C.H)), C.tan_half);
  d3 d = mk3(dadd(dadd(C.fwd[0], dmul(sx, C.right[0])), dmul(sy, C.up[0])),
             dadd(dadd(C.fwd[1], dmul(sx, C.right[1])), dmul(sy, C.up[1])),
             dadd(dadd(C.fwd[2], dmul(sx, C.right[2])), dmul(sy, C.up[2])));
  const double nr = norm3(d);
  d = mk3(ddiv(d.x, nr), ddiv(d.y, nr), ddiv(d.z, nr));
  const d3 o = mk3(C.pos[0], C.pos[1], C.pos[2]);
  st3(S.o, p, o);
  st3(S.d, p, d);
  S.thr[p] = 1.0;
  S.rad[p] = 0.0;
  S.alive[p] = 0;
  begin_trace(F, S, p, o, d);
}
#endif

// render.py:54-75 pixel_rays at pixel centres (offsets 0.5) for the
// single-bounce modes; slot p = pixel p
#ifndef DDF_OPS_ONLY
__global__ void camera_center_kernel(const FieldDev F, const CamDev C, const PathState S, int P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double px = (double)(p % C.W), py = (double)(p / C.W);
  const double sx = dmul(dmul(dsub(ddiv(dmul(2.0, dadd(px, 0.5)), (double)C.W), 1.0), C.tan_half), C.aspect);
  const double sy = dmul(dsub(1.0, ddiv(dmul(2.0, dadd(py, 0.5)), (double)C.H)), C.tan_half);
  d3 d = mk3(dadd(dadd(C.fwd[0], dmul(sx, C.right[0])), dmul(sy, C.up[0])),
             dadd(dadd(C.fwd[1], dmul(sx, C.right[1])), dmul(sy, C.up[1])),
             dadd(dadd(C.fwd[2], dmul(sx, C.right[2])), dmul(sy, C.up[2])));
  const double nr = norm3(d);
  d = mk3(ddiv(d.x, nr), ddiv(d.y, nr), ddiv(d.z, nr));
  const d3 o = mk3(C.pos[0], C.pos[1], C.pos[2]);
  st3(S.o, p, o);
  st3(S.d, p, d);
  begin_trace(F, S, p, o, d);
}
#endif

struct ModeDev {
  int mode, ambient;
  double bg[3], light[3], albedo, env;
};

// render.py:144-184 per pixel from the trace (t, hit) and, for hit pixels,
// the spatial gradient / face cross product in g3 (_hit_normals semantics)
#ifndef DDF_OPS_ONLY
__global__ void mode_shade_kernel(const ModeDev m, const PathState S, int P, double* out, int* err,
                                  unsigned long long* degenerate) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const bool h = S.hit[p];
  if (m.mode == 0) {
    out[p] = h ? S.t[p] : INFINITY;
    return;
  }
  double rgb[3] = {m.bg[0], m.bg[1], m.bg[2]};
  if (h) {
    const d3 d = ld3(S.d, p), g = ld3(S.g3, p);
    const double nr = norm3(g);
    d3 n;
    if (nr >= 1e-12) {
      n = mk3(ddiv(g.x, nr), ddiv(g.y, nr), ddiv(g.z, nr));
      if (dot3(n, d) > 0.0) n = mk3(-n.x, -n.y, -n.z);
    } else {
      n = mk3(-d.x, -d.y, -d.z);
      atomicAdd(degenerate, 1ull);
    }
    if (!(dot3(n, d) < 0.0)) atomicOr(err, (int)DEVERR_SIGN_RULE);
    if (m.mode == 1) {
      rgb[0] = dmul(0.5, dadd(n.x, 1.0));
      rgb[1] = dmul(0.5, dadd(n.y, 1.0));
      rgb[2] = dmul(0.5, dadd(n.z, 1.0));
    } else {
      const double c = m.ambient ? dmul(m.albedo, m.env)
                                 : dmul(m.albedo, fmax(dadd(dadd(dmul(n.x, m.light[0]), dmul(n.y, m.light[1])),
                                                            dmul(n.z, m.light[2])), 0.0));
      rgb[0] = rgb[1] = rgb[2] = c;
    }
  }
  out[3 * (int64_t)p] = rgb[0];
  out[3 * (int64_t)p + 1] = rgb[1];
  out[3 * (int64_t)p + 2] = rgb[2];
}
#endif

// render.py:218-219  escape of primary rays, alive = hit
#ifndef DDF_OPS_ONLY
__global__ void after_primary_kernel(const WaveDev w, const PathState S, int P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const bool h = S.hit[p];
  if (!h) S.rad[p] = w.env;
  S.alive[p] = h;
}
#endif

// EXTENSION (config 4): Russian roulette at bounce b >= rr_start,
// survival p = min(1, throughput), survivors divide by p.
__device__ __forceinline__ bool rr_survives(const WaveDev& w, double thr, int s, int i, int b, double& q) {
  q = fmin(1.0, thr);
  const double u = pcg_single(*w.rr, (uint64_t)(s * w.bounces + b) * (uint64_t)w.n_pix + (uint64_t)i);
  return u < q;
}
#ifndef DDF_OPS_ONLY
__global__ void roulette_kernel(const WaveDev w, const PathState S, int P, int b) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P || !S.alive[p]) return;
  int s, i;
  slot_sp(w, p, s, i);
  double q;
  if (rr_survives(w, S.thr[p], s, i, b, q)) S.thr[p] = ddiv(S.thr[p], q);
  else S.alive[p] = 0;
}
#endif

// field.py:103-112 orthonormal_frames + render.py:187-195 _cosine_dirs
__device__ __forceinline__ d3 cosine_dir(d3 n, double u0, double u1) {
  const double r = __dsqrt_rn(u0);
  const double phi = dmul(6.283185307179586, u1);
  const double l0 = dmul(r, cos(phi)), l1 = dmul(r, sin(phi));
  const double l2 = __dsqrt_rn(fmax(0.0, dsub(1.0, u0)));
  const double ax = fabs(n.x), ay = fabs(n.y), az = fabs(n.z);
  // np.argmin: first minimum
  int k = 0;
  double mn = ax;
  if (ay < mn) { k = 1; mn = ay; }
  if (az < mn) { k = 2; }
  const d3 axis = mk3(k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0);
  d3 t1 = cross3(n, axis);
  const double tn = norm3(t1);
  t1 = mk3(ddiv(t1.x, tn), ddiv(t1.y, tn), ddiv(t1.z, tn));
  const d3 t2 = cross3(n, t1);
  return mk3(dadd(dadd(dmul(l0, t1.x), dmul(l1, t2.x)), dmul(l2, n.x)),
             dadd(dadd(dmul(l0, t1.y), dmul(l1, t2.y)), dmul(l2, n.y)),
             dadd(dadd(dmul(l0, t1.z), dmul(l1, t2.z)), dmul(l2, n.z)));
}

// Gradient pass of a bounce (field.py:295-317 input, render.py:226): the
// MLP kernel evaluates d pred / d x at o + max(t - delta/2, 0) d with the
// stored angle inputs and writes the spatial gradient; bounce_kernel below
// turns it into the normal, hit point and next ray (memory-bound, off the
// tensor-core critical path).
struct GradOutOp : ListBase {
  static constexpr bool kGrad = true;
  static constexpr bool kRaw = false;
  PathState S; double backoff;
  __device__ double raw(int, int) const { return 0.0; }
  __device__ void load(int p, double* q, double& u3, double& u4) const {
    const d3 o = ld3(S.o, p), d = ld3(S.d, p);
    const double back = fmax(dsub(S.t[p], backoff), 0.0);
    q[0] = dadd(o.x, dmul(back, d.x)); q[1] = dadd(o.y, dmul(back, d.y)); q[2] = dadd(o.z, dmul(back, d.z));
    u3 = S.u34[2 * p];
    u4 = S.u34[2 * p + 1];
  }
  __device__ void store_grad(int p, const double* g5) const { st3(S.g3, p, mk3(g5[0], g5[1], g5[2])); }
  template <class G>
  __device__ void store_grad_raw(int, G) const {}
};

// Fused normal reuse: march step 0 of a bounce ray evaluates
// the network at o + t_acc d.  The next bounce's normal (field.py:305-309)
// evaluates it at o + max(t - delta/2, 0) d with the same angle inputs, so
// when the two f64 offsets are equal the inputs are identical bit for bit and
// one kernel can run the forward (distance, hit test, advance) and the
// backward chain on the same tile: the gradient is kept for exactly those
// rows (gdone = 1) and the gradient pass of the next bounce skips them.  The
// result equals the unfused path's: same program, same inputs, same order.
struct TraceGradOp : TraceStepOp {
  static constexpr bool kFused = true;
  double backoff; double* g3; uint8_t* gdone;
  __device__ void store_grad(int s, const double* g5) const {
    if (!st.hit[s]) return;
    if (st.t_acc[s] != fmax(dsub(st.t_out[s], backoff), 0.0)) return;
    st3(g3, s, mk3(g5[0], g5[1], g5[2]));
    gdone[s] = 1;
  }
  template <class G>
  __device__ void store_grad_raw(int, G) const {}
};

// normal + render.py:_hit_normals (127-141) + hit point, throughput, cosine
// bounce (render.py:226-231) + slab test of the new ray
#ifndef DDF_OPS_ONLY
__global__ void bounce_kernel(const FieldDev* F, const WaveDev w, const PathState S, const int* list,
                              const int* count, int b) {
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int p = list[k];
    const d3 o = ld3(S.o, p), d = ld3(S.d, p);
    const d3 g = ld3(S.g3, p);
    const double nr = norm3(g);                              // field.py:311-316
    d3 nn;
    if (nr >= 1e-12) {
      nn = mk3(ddiv(g.x, nr), ddiv(g.y, nr), ddiv(g.z, nr));
      if (dot3(nn, d) > 0.0) nn = mk3(-nn.x, -nn.y, -nn.z);
    } else {
      nn = mk3(-d.x, -d.y, -d.z);                            // render.py:133-136
      atomicAdd(w.degenerate, 1ull);
    }
    if (!(dot3(nn, d) < 0.0)) atomicOr(w.err, (int)DEVERR_SIGN_RULE);   // render.py:137-139
    const double t = S.t[p];
    const d3 hp = mk3(dadd(dadd(o.x, dmul(t, d.x)), dmul(1e-6, nn.x)),
                      dadd(dadd(o.y, dmul(t, d.y)), dmul(1e-6, nn.y)),
                      dadd(dadd(o.z, dmul(t, d.z)), dmul(1e-6, nn.z)));
    const int ob = S.obj[p];
    S.thr[p] = dmul(S.thr[p], F->composite ? F->net[ob].albedo : w.albedo);
    int s, i;
    slot_sp(w, p, s, i);
    double u0, u1;
    pcg_pair(*w.rng, (uint64_t)(s * (w.bounces + 1) + 1 + b) * 2ull * (uint64_t)w.n_pix + 2ull * (uint64_t)i, u0, u1);
    const d3 nd = cosine_dir(nn, u0, u1);
    st3(S.o, p, hp);
    st3(S.d, p, nd);
    begin_trace(*F, S, p, hp, nd);
    if (S.want) {
      // fused normal reuse: the next bounce needs this segment's normal only
      // if there is a next bounce and the path survives its roulette (same
      // draw and throughput roulette_kernel will see); the first march input
      // can equal the normal input only for t_acc == 0
      bool want = b + 1 < w.bounces && S.march[p] && S.t_acc[p] == 0.0;
      if (want && w.rr_start >= 0 && b + 1 >= w.rr_start) {
        double q;
        want = rr_survives(w, S.thr[p], s, i, b + 1, q);
      }
      S.want[p] = want;
    }
  }
}
#endif

// render.py:233-242 over the bounce's alive list
#ifndef DDF_OPS_ONLY
__global__ void after_bounce_kernel(const WaveDev w, const PathState S, const int* list, const int* count) {
  const int n = *count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int p = list[k];
    if (!S.hit[p]) {
      S.rad[p] = dadd(S.rad[p], dmul(S.thr[p], w.env));
      S.alive[p] = 0;
    }
  }
}
#endif

// render.py:243  accum += radiance, in sample order
#ifndef DDF_OPS_ONLY
__global__ void film_kernel(const WaveDev w, const PathState S, double* accum) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= w.n_own) return;
  const int i = w.pix[q];
  double a = accum[i];
  for (int s = 0; s < w.ns; ++s) a = dadd(a, S.rad[(int64_t)s * w.n_own + q]);
  accum[i] = a;
}
#endif

}  // namespace ddf
