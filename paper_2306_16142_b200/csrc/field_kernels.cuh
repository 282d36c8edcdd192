// Field-level kernels: one persistent kernel per MLP pass, parameterised by a
// row operation ("Op") that says where each row's ray comes from and what to
// do with the prediction / gradient.  The same Ops drive the fp32 SIMT engine
// (here) and the bf16 tcgen05 engine (mlp_umma.cuh).
//
// Row ops restate, per row, the reference's numpy batch code:
//   RawForwardOp  neural.forward_batch        neural.py:138-157
//   RawGradOp     neural.input_gradient_batch neural.py:229-249
//   QueryOp       NeuralField.query_batch     field.py:248-258
//   TraceStepOp   one step of trace_batch     field.py:274-288
//   NormalOp      NeuralField.normal_batch    field.py:295-317
// (GradOutOp, the gradient pass of render_path's bounce stage, lives in
// wavefront.cuh.)
#pragma once
#include "ddf_common.cuh"
#include "mlp_simt.cuh"

namespace ddf {

// ---------------------------------------------------------------- encoding
// Network input k (padded width) of one row from its 5 encoded values u.
// PE layout (EXTENSION, configs 3-5): [u0..u4, {sin(2^o pi u), cos(2^o pi u)} o=0..5]
__device__ __forceinline__ double input_value(const NetDev& net, const double u[5], int k) {
  if (k < 5) return u[k];
  if (net.encoding != ENC_PE6 || k >= 5 + 10 * DDF_PE_OCTAVES) return 0.0;
  const int o = (k - 5) / 10, r = (k - 5) % 10;
  const double f = (double)(1 << o) * 3.141592653589793;   // (2.0**o)*np.pi, exact power-of-2 scale
  return r < 5 ? sin(dmul(f, u[r])) : cos(dmul(f, u[r - 5]));
}

// chain rule through the PE (oracle/cpu_ddf.py pe_chain); g has the padded input width
template <class G>
__device__ __forceinline__ void pe_chain(const NetDev& net, const double u[5], G g, double out[5]) {
  for (int j = 0; j < 5; ++j) out[j] = g(j);
  if (net.encoding != ENC_PE6) return;
  for (int o = 0; o < DDF_PE_OCTAVES; ++o) {
    const double f = (double)(1 << o) * 3.141592653589793;
    for (int j = 0; j < 5; ++j) {
      const double a = dmul(f, u[j]);
      out[j] = dadd(out[j], dmul(dmul(f, cos(a)), g(5 + 10 * o + j)));
      out[j] = dsub(out[j], dmul(dmul(f, sin(a)), g(5 + 10 * o + 5 + j)));
    }
  }
}

// per-row encoded inputs (before PE) for object j: composite fields see
// (p - c_j) / s (EXTENSION, config 5); single nets see p (neural.py:35-37).
// Row ops hand over the two encoded angle inputs u3 = az/pi - 1,
// u4 = 2 pol/pi - 1 (neural.py:36-37) already computed.
__device__ __forceinline__ void row_u(const FieldDev& F, int j, const double* pos, double u3, double u4,
                                      double u[5]) {
  if (F.composite) {
    const NetDev& n = F.net[j];
    for (int c = 0; c < 3; ++c) u[c] = ddiv(dsub(pos[c], n.center[c]), n.scale);
  } else {
    for (int c = 0; c < 3; ++c) u[c] = pos[c];
  }
  u[3] = u3;
  u[4] = u4;
}

// The same for the bf16 engines: the object-local position by a multiply with
// 1 / scale instead of three f64 divisions (one f64 ulp apart, far below the
// bf16 rounding of the encoded inputs).  The divisions were a measurable part
// of the ~2 K-cycle encoding at each of config 5's eight network boundaries
// per tile; the fp32 engines keep row_u.
__device__ __forceinline__ void row_u_bf16(const FieldDev& F, int j, const double* pos, double u3, double u4,
                                           double u[5]) {
  if (F.composite) {
    const NetDev& n = F.net[j];
    for (int c = 0; c < 3; ++c) u[c] = dmul(dsub(pos[c], n.center[c]), n.inv_scale);
  } else {
    for (int c = 0; c < 3; ++c) u[c] = pos[c];
  }
  u[3] = u3;
  u[4] = u4;
}

// encoded angle inputs of a unit direction (field.py:77-82 + neural.py:36-37)
__device__ __forceinline__ void dir_u34(d3 d, double& u3, double& u4) {
  double az, pol;
  dir_angles(d, az, pol);
  encode_angles(az, pol, u3, u4);
}

// Encoded angle inputs of a query direction the way query_batch forms them:
// vecs_to_angles (field.py:258), then _predict's re-canonicalisation
// angles -> unit vector -> angles (field.py:251).  Away from the poles and
// the azimuth wrap the second pass returns the first pass's angles to within
// a few f64 ulps (it exists to canonicalise az at the poles and at 0 = 2 pi),
// far below the fp32 / tf32-split / bf16 rounding every engine applies to the
// inputs; there the first pass is used directly.  That halves the f64
// trigonometry per ray (2 atan2 + 2 acos + 2 sincos -> 1 + 1), which bounded
// the <= 128-wide query: ~9 K of 25 K cycles per 512-row pack.  Near a pole
// (sin pol < 1e-3) or the wrap (az within 1e-6 of 0 or 2 pi) the reference's
// exact sequence runs.
__device__ __forceinline__ void query_dir_u34(d3 d, double& u3, double& u4) {
  double a0, a1;
  dir_angles(d, a0, a1);
  const double two_pi = 6.283185307179586;
  const bool edge = !(a1 > 1e-3 && a1 < 3.1405926535897933 && a0 > 1e-6 && a0 < two_pi - 1e-6);
  if (edge) dir_u34(angles_dir(a0, a1), u3, u4);
  else encode_angles(a0, a1, u3, u4);
}

__device__ __forceinline__ d3 ld3(const double* a, int64_t i) { return mk3(a[3 * i], a[3 * i + 1], a[3 * i + 2]); }
__device__ __forceinline__ void st3(double* a, int64_t i, d3 v) { a[3 * i] = v.x; a[3 * i + 1] = v.y; a[3 * i + 2] = v.z; }

// ---------------------------------------------------------------- row ops
struct ListBase {
  static constexpr bool kFused = false;   // true: trace step + input gradient in one pass (TraceGradOp)
  const int* list;      // slot ids (nullptr = identity)
  const int* count;     // device count (nullptr = n)
  int n;
  const int* seg;       // [n_obj+1] segment offsets into list for gradient passes (nullptr = one segment)
  __device__ int total() const { return count ? *count : n; }
  __device__ int slot(int i) const { return list ? list[i] : i; }
  __device__ int seg_begin(int j) const { return seg ? seg[j] : (j == 0 ? 0 : total()); }
  __device__ int seg_end(int j) const { return seg ? seg[j + 1] : total(); }
};

struct RawForwardOp : ListBase {
  static constexpr bool kGrad = false;
  static constexpr bool kRaw = true;
  const double* x; int width; double* out;
  __device__ double raw(int s, int k) const { return k < width ? x[(int64_t)s * width + k] : 0.0; }
  __device__ void load(int, double*, double&, double&) const {}
  __device__ void store_fwd(int s, double pred, int) const { out[s] = pred; }
};

struct RawGradOp : ListBase {
  static constexpr bool kGrad = true;
  static constexpr bool kRaw = true;
  const double* x; int width; double* out;
  __device__ double raw(int s, int k) const { return k < width ? x[(int64_t)s * width + k] : 0.0; }
  __device__ void load(int, double*, double&, double&) const {}
  template <class G>
  __device__ void store_grad_raw(int s, G g) const {
    for (int k = 0; k < width; ++k) out[(int64_t)s * width + k] = g(k);
  }
  __device__ void store_grad(int, const double*) const {}
};

struct QueryOp : ListBase {
  static constexpr bool kGrad = false;
  static constexpr bool kRaw = false;
  const double* pos; const double* dirs;
  double* t; uint8_t* hit; double* pred_out; int* obj_out;
  double delta, thresh;
  __device__ double raw(int, int) const { return 0.0; }
  __device__ void load(int s, double* p, double& u3, double& u4) const {
    const d3 q = ld3(pos, s);
    p[0] = q.x; p[1] = q.y; p[2] = q.z;
    query_dir_u34(ld3(dirs, s), u3, u4);
  }
  __device__ void store_fwd(int s, double pred, int obj) const {
    const double c = fmin(fmax(pred, -delta), delta);   // field.py:253
    t[s] = fmax(c, 0.0);
    hit[s] = c < thresh;
    if (pred_out) pred_out[s] = pred;
    if (obj_out) obj_out[s] = obj;
  }
};

// Ray state of the sphere march (field.py:265-288), SoA in HBM.
struct MarchState {
  const double* o; const double* d;   // (n,3) origins / unit directions
  double* t_acc; const double* t_exit;
  uint8_t* alive; double* t_out; uint8_t* hit; int* obj;
  const double* u34;                  // (n,2) encoded angles of d, or nullptr (computed per step)
};

struct TraceStepOp : ListBase {
  static constexpr bool kGrad = false;
  static constexpr bool kRaw = false;
  MarchState st; double delta, thresh, step;
  __device__ double raw(int, int) const { return 0.0; }
  __device__ void load(int s, double* p, double& u3, double& u4) const {
    const d3 o = ld3(st.o, s), d = ld3(st.d, s);
    const double ta = st.t_acc[s];
    p[0] = dadd(o.x, dmul(ta, d.x)); p[1] = dadd(o.y, dmul(ta, d.y)); p[2] = dadd(o.z, dmul(ta, d.z));
    if (st.u34) { u3 = st.u34[2 * s]; u4 = st.u34[2 * s + 1]; }
    else dir_u34(d, u3, u4);
  }
  __device__ void store_fwd(int s, double pred, int obj) const {
    const double c = fmin(fmax(pred, -delta), delta);
    if (c < thresh) {                                       // field.py:281-285
      st.t_out[s] = dadd(st.t_acc[s], fmax(c, 0.0));
      st.hit[s] = 1;
      st.obj[s] = obj;
      st.alive[s] = 0;
    } else {                                                // field.py:286-288
      const double ta = dadd(st.t_acc[s], step);
      st.t_acc[s] = ta;
      if (ta > st.t_exit[s]) st.alive[s] = 0;
    }
  }
};

struct NormalOp : ListBase {
  static constexpr bool kGrad = true;
  static constexpr bool kRaw = false;
  const double* o; const double* d; const double* t_hit;  // t_hit nullable
  double backoff; double* normals; uint8_t* valid;
  __device__ double raw(int, int) const { return 0.0; }
  __device__ void load(int s, double* p, double& u3, double& u4) const {
    const d3 oo = ld3(o, s), dd = ld3(d, s);
    if (t_hit) {                                            // field.py:305-307
      const double back = fmax(dsub(t_hit[s], backoff), 0.0);
      p[0] = dadd(oo.x, dmul(back, dd.x)); p[1] = dadd(oo.y, dmul(back, dd.y)); p[2] = dadd(oo.z, dmul(back, dd.z));
    } else {
      p[0] = oo.x; p[1] = oo.y; p[2] = oo.z;
    }
    dir_u34(dd, u3, u4);
  }
  __device__ void store_grad(int s, const double* g5) const {
    const d3 g = mk3(g5[0], g5[1], g5[2]);                  // field.py:310-316
    const double nr = norm3(g);
    const bool ok = nr >= 1e-12;
    d3 n = ok ? mk3(ddiv(g.x, nr), ddiv(g.y, nr), ddiv(g.z, nr)) : mk3(0.0, 0.0, 0.0);
    if (dot3(n, ld3(d, s)) > 0.0) n = mk3(-n.x, -n.y, -n.z);
    st3(normals, s, n);
    valid[s] = ok;
  }
  template <class G>
  __device__ void store_grad_raw(int, G) const {}
};

// ---------------------------------------------------------------- fp32 engine kernels
namespace simt {

template <int M, int KMAX>
struct Tile {
  float* actA; float* actB; float* ws; float* head; uint32_t* mask;
  double* pos; double* ang; double* best; int* bobj; int* slot;
  __device__ static Tile carve(void* raw) {
    Tile t;
    char* p = reinterpret_cast<char*>(raw);
    t.pos = reinterpret_cast<double*>(p); p += sizeof(double) * M * 3;
    t.ang = reinterpret_cast<double*>(p); p += sizeof(double) * M * 2;
    t.best = reinterpret_cast<double*>(p); p += sizeof(double) * M * 3;
    t.actA = reinterpret_cast<float*>(p); p += sizeof(float) * KMAX * M;
    t.actB = reinterpret_cast<float*>(p); p += sizeof(float) * KMAX * M;
    t.ws = reinterpret_cast<float*>(p); p += sizeof(float) * 2 * KC * NC;   // double-buffered weight chunks
    t.head = reinterpret_cast<float*>(p); p += sizeof(float) * M * 2;
    t.mask = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * DDF_MAX_LAYERS * KMAX * (M / 32);
    t.bobj = reinterpret_cast<int*>(p); p += sizeof(int) * M;
    t.slot = reinterpret_cast<int*>(p);
    return t;
  }
};

template <int M, int KMAX, class Op>
__device__ __forceinline__ void fill_inputs(const FieldDev& F, int j, const Op& op, const Tile<M, KMAX>& T,
                                            int nv) {
  const NetDev& net = F.net[j];
  const int K0 = net.widths[0];
  for (int idx = threadIdx.x; idx < K0 * M; idx += NT) {
    const int k = idx / M, m = idx % M;
    double v = 0.0;
    if (m < nv) {
      if constexpr (Op::kRaw) {
        v = op.raw(T.slot[m], k);
      } else {
        double u[5];
        row_u(F, j, T.pos + 3 * m, T.ang[2 * m], T.ang[2 * m + 1], u);
        v = input_value(net, u, k);
      }
    }
    T.actA[k * M + m] = (float)v;
  }
  __syncthreads();
}

template <int M, int KMAX, class Op>
__device__ __forceinline__ void load_rows(const Op& op, const Tile<M, KMAX>& T, int base, int nv) {
  if (threadIdx.x < M) {
    const int m = threadIdx.x;
    if (m < nv) {
      const int s = op.slot(base + m);
      T.slot[m] = s;
      double az = 0.0, pol = 0.0;
      op.load(s, T.pos + 3 * m, az, pol);
      T.ang[2 * m] = az;
      T.ang[2 * m + 1] = pol;
    }
  }
  __syncthreads();
}

// forward over all objects, min-composite (EXTENSION for > 1 object)
template <int M, int KMAX, class Op>
__global__ void __launch_bounds__(NT) forward_kernel(const FieldDev F, const Op op) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Tile<M, KMAX> T = Tile<M, KMAX>::carve(smem_raw);
  const int n = op.total();
  for (int base = blockIdx.x * M; base < n; base += gridDim.x * M) {
    const int nv = min(M, n - base);
    load_rows<M, KMAX>(op, T, base, nv);
    for (int j = 0; j < F.n_obj; ++j) {
      const NetDev& net = F.net[j];
      fill_inputs<M, KMAX>(F, j, op, T, nv);
      float* a = T.actA;
      float* b = T.actB;
      const int L = net.n_layers;
      for (int l = 0; l < L - 1; ++l) {
        gemm_layer<M>(net.wt[l], net.b[l], net.widths[l], net.widths[l + 1], a, b, T.ws, EPI_RELU, nullptr, nullptr);
        float* t = a; a = b; b = t;
      }
      // head bias is read from device memory (fp32)
      head_dot<M>(net.w[L - 1], __ldg(net.b[L - 1]), net.widths[L - 1], a, T.head);
      if (threadIdx.x < nv) {
        double p = (double)T.head[threadIdx.x];
        if (F.composite) p = dmul(net.scale, p);
        if (j == 0 || p < T.best[threadIdx.x]) { T.best[threadIdx.x] = p; T.bobj[threadIdx.x] = j; }
      }
      __syncthreads();
    }
    if (threadIdx.x < nv) op.store_fwd(T.slot[threadIdx.x], T.best[threadIdx.x], T.bobj[threadIdx.x]);
    __syncthreads();
  }
}

// input gradient of object j's network for the rows of segment j
template <int M, int KMAX, class Op>
__global__ void __launch_bounds__(NT) grad_kernel(const FieldDev F, const Op op) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Tile<M, KMAX> T = Tile<M, KMAX>::carve(smem_raw);
  // enumerate (object, tile) pairs over the segments
  int tiles_before[DDF_MAX_OBJECTS + 1];
  tiles_before[0] = 0;
  for (int j = 0; j < F.n_obj; ++j) {
    const int c = op.seg_end(j) - op.seg_begin(j);
    tiles_before[j + 1] = tiles_before[j] + (c + M - 1) / M;
  }
  const int n_tiles = tiles_before[F.n_obj];
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    int j = 0;
    while (tile >= tiles_before[j + 1]) ++j;
    const int base = op.seg_begin(j) + (tile - tiles_before[j]) * M;
    const int nv = min(M, op.seg_end(j) - base);
    const NetDev& net = F.net[j];
    const int L = net.n_layers;
    load_rows<M, KMAX>(op, T, base, nv);
    for (int i = threadIdx.x; i < DDF_MAX_LAYERS * KMAX * (M / 32); i += NT) T.mask[i] = 0u;
    fill_inputs<M, KMAX>(F, j, op, T, nv);
    float* a = T.actA;
    float* b = T.actB;
    const int mstride = KMAX * (M / 32);
    for (int l = 0; l < L - 1; ++l) {
      gemm_layer<M>(net.wt[l], net.b[l], net.widths[l], net.widths[l + 1], a, b, T.ws, EPI_RELU_MASK,
                    T.mask + l * mstride, nullptr);
      float* t = a; a = b; b = t;
    }
    // d/dh of the head = w_head, masked by the last hidden layer (neural.py:244-247)
    {
      const int H = net.widths[L - 1];
      const float* wh = net.w[L - 1];
      const uint32_t* mk = (L >= 2) ? T.mask + (L - 2) * mstride : nullptr;
      for (int idx = threadIdx.x; idx < H * M; idx += NT) {
        const int k = idx / M, m = idx % M;
        float v = __ldg(wh + k);
        if (mk && !((mk[k * (M / 32) + (m >> 5)] >> (m & 31)) & 1u)) v = 0.f;
        a[k * M + m] = v;
      }
      __syncthreads();
    }
    for (int l = L - 2; l >= 0; --l) {
      gemm_layer<M>(net.w[l], nullptr, net.widths[l + 1], net.widths[l], a, b, T.ws,
                    l > 0 ? EPI_MASKMUL : EPI_LINEAR, nullptr, l > 0 ? T.mask + (l - 1) * mstride : nullptr);
      float* t = a; a = b; b = t;
    }
    if (threadIdx.x < nv) {
      const int m = threadIdx.x;
      if constexpr (Op::kRaw) {
        op.store_grad_raw(T.slot[m], [&](int k) { return (double)a[k * M + m]; });
      } else {
        double u[5], g5[5];
        row_u(F, j, T.pos + 3 * m, T.ang[2 * m], T.ang[2 * m + 1], u);
        pe_chain(net, u, [&](int k) { return (double)a[k * M + m]; }, g5);
        op.store_grad(T.slot[m], g5);
      }
    }
    __syncthreads();
  }
}

}  // namespace simt
}  // namespace ddf
