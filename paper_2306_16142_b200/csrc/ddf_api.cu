// libddf_b200.so: the C ABI (include/ddf_b200.h) over the sm_100a kernels.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ddf_b200.h"
#include "compact.cuh"
#include "engines.h"
#include "ddf_common.cuh"
#include "field_kernels.cuh"
#include "mlp_umma.cuh"
#include "mlp_x3.cuh"
#include "udf.cuh"
#include "mesh.cuh"
#include "wavefront.cuh"

using namespace ddf;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) return fail(DDF_ECUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

int pad16(int w) { return (w + 15) / 16 * 16; }

// bumped whenever any scratch buffer moves: captured render graphs hold raw
// buffer pointers and are keyed by it
unsigned long long g_buf_epoch = 0;

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    ++g_buf_epoch;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

}  // namespace

// Per-call kernel-class timing (cfg->profile) and launch counting.
struct Prof {
  // OTHER = the wavefront kernels, split per kernel for the HBM roofline
  enum { FWD = 0, GRAD = 1, COMPACT = 2, OTHER = 3, TOTAL = 4, FUSED = 5, CAMERA = 6, ROULETTE = 7, BOUNCE = 8,
         AFTER = 9, FILM = 10, NCAT = 11 };
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<size_t, size_t>> marks[NCAT];
  uint64_t launches = 0, fwd_launches = 0, grad_launches = 0, fused_launches = 0;
  void reset(bool enable) {
    on = enable;
    used = 0;
    for (auto& m : marks) m.clear();
    launches = fwd_launches = grad_launches = fused_launches = 0;
  }
  size_t rec(cudaStream_t st) {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    cudaEventRecord(pool[used], st);
    return used++;
  }
  double total_ms(int cat) {
    double t = 0.0;
    for (auto& m : marks[cat]) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pool[m.first], pool[m.second]);
      t += ms;
    }
    return t;
  }
};

struct ddf_field_s {
  Prof prof;
  FieldDev F{};                 // host copy holding device pointers
  FieldDev* F_dev = nullptr;    // device copy (bounce_kernel reads albedos through it)
  std::vector<void*> weights;   // device weight allocations
  std::vector<umma::NetImage> images;
  std::vector<umma::NetImage> images_x3;   // 3xTF32 images (empty entries for networks the engine cannot take)
  int device = 0;
  int sm_count = 148;
  // scratch
  Buf t_acc, t_exit, alive, list, list2, blocks, small, ones;
  Buf op_state;   // single-pass compaction state: zero between calls (compact.cuh onepass_kernel)
  Buf st_o, st_d, st_tacc, st_texit, st_t, st_thr, st_rad, st_hit, st_march, st_alive, st_obj;
  Buf pix, rng, umma_masks, st_u34, st_g3, st_gdone, st_want;
  Buf film;   // the render's accumulator: captured graphs write here, the caller's buffer gets a copy
  Buf udf_dirs, udf_vals, udf_pts, udf_best, udf_arg, udf_found, udf_list, udf_seg, udf_state;
  // captured render_path waves (cfg->graph): replayed while the key matches
  unsigned long long gen = 0;            // bumped by add_network / set_precision
  cudaStream_t cap_stream = nullptr;     // private capture stream
  cudaGraphExec_t graph_exec = nullptr;
  std::vector<unsigned char> graph_key;
  int graph_waves = 0;
  uint64_t graph_launches[4] = {0, 0, 0, 0};
  // exact mesh field (ddf_mesh_create)
  mesh::MeshDev M{};
  Buf mesh_nodes, mesh_tris, mesh_tof;
  int udf_ndirs = 0;
  int pix_key[6] = {-1, -1, -1, -1, -1, -1};
  std::vector<int32_t> pix_owner;        // cfg->tile_owner the cached pixel list was built from
  int pix_n = 0;
};

namespace {

// small scratch layout: [0..15] seg, [16] count, [17] count2, [18..19] err, u64 stats after 32 ints:
// [0] forward rows, [1] gradient rows (reference count: rows needing a normal),
// [2] degenerate normals, [3] fused trace+gradient rows, [4] rows of the
// gradient pass proper when fusion is on
// [16..) per-stage rows: primary march steps [16, 80), bounce alive [80, 112), bounce march [112, 144)
struct Small {
  int* seg; int* count; int* count2; int* err; unsigned long long* stats;  // stats[0]=fwd [1]=grad [2]=degenerate
  unsigned long long* primary_rows() const { return stats + 16; }
  unsigned long long* alive_rows() const { return stats + 16 + DDF_STAGE_STEPS; }
  unsigned long long* bmarch_rows() const { return stats + 16 + DDF_STAGE_STEPS + DDF_STAGE_BOUNCES; }
};
constexpr int SMALL_U64 = 16 + DDF_STAGE_STEPS + 2 * DDF_STAGE_BOUNCES;   // u64 stats words in use
Small small_of(ddf_field_s* f) {
  Small s;
  int* b = f->small.as<int>();
  s.seg = b;
  s.count = b + 16;
  s.count2 = b + 17;
  s.err = b + 18;
  s.stats = reinterpret_cast<unsigned long long*>(b + 32);
  return s;
}

int max_width(const FieldDev& F) {
  int w = 0;
  for (int j = 0; j < F.n_obj; ++j)
    for (int l = 0; l <= F.net[j].n_layers; ++l) w = std::max(w, F.net[j].widths[l]);
  return w;
}

// ---------------------------------------------------------------- engine dispatch
// RAII marker: records start/stop events of one kernel-class region
struct ProfScope {
  Prof& p; int cat; cudaStream_t st; size_t a = 0;
  ProfScope(Prof& p_, int c, cudaStream_t s) : p(p_), cat(c), st(s) { if (p.on) a = p.rec(st); }
  ~ProfScope() { if (p.on) p.marks[cat].push_back({a, p.rec(st)}); }
};

template <class Op>
int run_mlp(ddf_field_s* f, const FieldDev& F, const Op& op, int max_rows, bool grad, cudaStream_t st) {
  if (max_rows <= 0) return DDF_OK;
  ProfScope ps(f->prof, grad ? Prof::GRAD : Prof::FWD, st);
  f->prof.launches += 1;
  (grad ? f->prof.grad_launches : f->prof.fwd_launches) += 1;
  // fp32 mode: the 3xTF32 tensor-core engine when every network fits it
  bool x3 = F.precision == PREC_FP32;
  for (int j = 0; j < F.n_obj; ++j) x3 = x3 && F.net[j].wimg_x3 != nullptr;
  if (x3) {
    CUDA_TRY(f->umma_masks.ensure(sizeof(uint32_t) * (size_t)umma::MASK_WORDS_PER_CTA * umma::QS * f->sm_count));
    std::vector<umma::NetImage> imgs;
    if (F.n_obj == 1 && f->F.n_obj > 1) {
      for (auto& im : f->images_x3)
        if (im.dev == F.net[0].wimg_x3) imgs.push_back(im);
    } else {
      imgs = f->images_x3;
    }
    int rc = engines::x3_launch<Op>(F, imgs, op, max_rows, f->sm_count, f->umma_masks.as<uint32_t>(), st, &g_err);
    return rc ? (rc == 1 ? DDF_EUSAGE : DDF_ECUDA) : DDF_OK;
  }
  bool tensor = F.precision == PREC_BF16;
  for (int j = 0; j < F.n_obj; ++j) tensor = tensor && F.net[j].wimg_fwd != nullptr;
  if (tensor) {
    CUDA_TRY(f->umma_masks.ensure(sizeof(uint32_t) * (size_t)umma::MASK_WORDS_PER_CTA * umma::QS * f->sm_count));
    std::vector<umma::NetImage> imgs;
    if (F.n_obj == 1 && f->F.n_obj > 1) {
      // single-network pass (ddf_mlp_*): find which image F.net[0] is
      for (auto& im : f->images)
        if (im.dev == F.net[0].wimg_fwd) imgs.push_back(im);
    } else {
      imgs = f->images;
    }
    int rc = engines::umma_launch<Op>(F, imgs, op, max_rows, f->sm_count, f->umma_masks.as<uint32_t>(), st, &g_err);
    return rc ? (rc == 1 ? DDF_EUSAGE : DDF_ECUDA) : DDF_OK;
  }
  const int rc = engines::simt_launch<Op>(F, op, max_rows, max_width(F), f->sm_count, st, &g_err);
  return rc ? (rc == 1 ? DDF_EUSAGE : DDF_ECUDA) : DDF_OK;
}

// Fused trace step + input gradient (TraceGradOp, wavefront.cuh) on the
// bf16 tcgen05 engine: one network wider than 256, single-step march regime
// (0.9 delta covers the box diagonal, so a bounce ray's step-0 input is where
// its normal will be evaluated).  Anything else keeps the unfused passes.
bool fusion_ok(const ddf_field_s* f) {
  const FieldDev& F = f->F;
  if (F.is_mesh || F.n_obj != 1 || F.composite || F.precision != PREC_BF16) return false;
  if (f->images.size() != 1 || !f->images[0].dev || f->images[0].host.pp) return false;
  double d2 = 0.0;
  for (int k = 0; k < 3; ++k) d2 += (F.hi[k] - F.lo[k]) * (F.hi[k] - F.lo[k]);
  return F.step >= std::sqrt(d2);
}

int run_fused(ddf_field_s* f, const TraceGradOp& op, int max_rows, cudaStream_t st) {
  if (max_rows <= 0) return DDF_OK;
  ProfScope ps(f->prof, Prof::FUSED, st);
  f->prof.launches += 1;
  f->prof.fused_launches += 1;
  CUDA_TRY(f->umma_masks.ensure(sizeof(uint32_t) * (size_t)umma::MASK_WORDS_PER_CTA * umma::QS * f->sm_count));
  int rc = engines::umma_launch<TraceGradOp>(f->F, f->images, op, max_rows, f->sm_count, f->umma_masks.as<uint32_t>(), st,
                                     &g_err);
  return rc ? (rc == 1 ? DDF_EUSAGE : DDF_ECUDA) : DDF_OK;
}

// stable compaction flags -> list (+ segments by object when obj != nullptr)
int compact_flags(ddf_field_s* f, const uint8_t* flags, const int* obj, int n, int n_obj, int* list, int* seg,
                  int* count, unsigned long long* rows_acc, cudaStream_t st, const uint8_t* sel = nullptr,
                  int sel_val = 0, unsigned long long* rows_acc2 = nullptr, unsigned long long* rows_acc3 = nullptr) {
  const int nb = std::max(1, (n + compact::BLOCK_ITEMS - 1) / compact::BLOCK_ITEMS);
  CUDA_TRY(f->blocks.ensure(sizeof(int) * nb * DDF_MAX_OBJECTS));
  int* bc = f->blocks.as<int>();
  const int no = obj ? n_obj : 1;
  ProfScope ps(f->prof, Prof::COMPACT, st);
  if (no == 1) {   // one segment: single pass with decoupled look-back
    const int nb1 = std::max(1, (n + compact::OP_ITEMS - 1) / compact::OP_ITEMS);
    // the kernel's own state buffer, zeroed when (re)allocated and left zero by every call
    const size_t sbytes = sizeof(unsigned long long) * (nb1 + compact::OP_STATE_EXTRA);
    if (sbytes > f->op_state.bytes) {
      CUDA_TRY(f->op_state.ensure(std::max(sbytes, (size_t)16384)));
      CUDA_TRY(cudaMemsetAsync(f->op_state.p, 0, f->op_state.bytes, st));
    }
    unsigned long long* state = f->op_state.as<unsigned long long>();
    f->prof.launches += 1;
    compact::onepass_kernel<<<nb1, compact::NT, 0, st>>>(flags, sel, sel_val, n, nb1, state, list, seg, count,
                                                          rows_acc, rows_acc2, rows_acc3);
    CUDA_TRY(cudaGetLastError());
    return DDF_OK;
  }
  f->prof.launches += 3;
  compact::count_kernel<<<nb, compact::NT, 0, st>>>(flags, sel, sel_val, obj, n, no, bc);
  compact::scan_kernel<<<1, 1024, 0, st>>>(bc, nb, no, seg, count, rows_acc, rows_acc2, rows_acc3);
  compact::scatter_kernel<<<nb, compact::NT, 0, st>>>(flags, sel, sel_val, obj, n, no, bc, list);
  CUDA_TRY(cudaGetLastError());
  return DDF_OK;
}

__global__ void trace_init_kernel(const FieldDev F, MarchState S, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const d3 o = ld3(S.o, i), d = ld3(S.d, i);
  double te, tx;
  ray_box(o, d, F.lo, F.hi, te, tx);
  const bool in = (te < tx) && (tx > 0.0);
  S.t_acc[i] = in ? fmax(te, 0.0) : 0.0;
  const_cast<double*>(S.t_exit)[i] = tx;
  S.alive[i] = in;
  S.t_out[i] = INFINITY;
  S.hit[i] = 0;
  if (S.obj) S.obj[i] = 0;
}

// stage log (ddf_path_config_t.stage_log): appends one compacted list as
// {kind, bounce, step, s0, n_own, count, ids...}.  Every block reads the same
// header word; the commit kernel that follows advances it.
struct StageLog {
  int* log = nullptr;
  long long cap = 0;
  int s0 = 0, n_own = 0;
};

__global__ void stage_log_copy_kernel(int* __restrict__ log, long long cap, const int* __restrict__ list,
                                      const int* __restrict__ count, int kind, int bounce, int step, int s0,
                                      int n_own) {
  const long long used = log[0];
  const int n = *count;
  if (log[1] || 2 + used + 6 + n > cap) return;
  int* rec = log + 2 + used;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rec[0] = kind; rec[1] = bounce; rec[2] = step; rec[3] = s0; rec[4] = n_own; rec[5] = n;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rec[6 + i] = list[i];
}

__global__ void stage_log_commit_kernel(int* log, long long cap, const int* count) {
  const long long need = 6 + (long long)*count;
  if (log[1] || 2 + (long long)log[0] + need > cap) log[1] = 1;
  else log[0] += (int)need;
}

int stage_log(ddf_field_s* f, const StageLog* lg, const int* list, const int* count, int kind, int bounce, int step,
              cudaStream_t st) {
  if (!lg || !lg->log) return DDF_OK;
  stage_log_copy_kernel<<<2 * f->sm_count, 256, 0, st>>>(lg->log, lg->cap, list, count, kind, bounce, step, lg->s0,
                                                         lg->n_own);
  stage_log_commit_kernel<<<1, 1, 0, st>>>(lg->log, lg->cap, count);
  f->prof.launches += 2;
  CUDA_TRY(cudaGetLastError());
  return DDF_OK;
}

// sphere march over the slots whose `march` flag is set (field.py:274-288)
// fused (nullable): step 0 of the rows whose `want` byte is set runs as
// TraceGradOp (fused normal reuse); the other rows take the plain step.
// step_rows (nullable): per-stage row counters, entry step * step_stride
// (stride 1: one counter per march step; 0: one counter for the whole march,
// ddf_render_stats_t.primary_march_rows / bounce_march_rows).  lg / bounce:
// the stage log (kind 0 for bounce < 0, else kinds 2 and 3).
int march(ddf_field_s* f, const MarchState& ms, int n, int* list, unsigned long long* fwd_acc, cudaStream_t st,
          const TraceGradOp* fused = nullptr, const uint8_t* want = nullptr,
          unsigned long long* step_rows = nullptr, int step_stride = 0, const StageLog* lg = nullptr,
          int bounce = -1) {
  Small sm = small_of(f);
  for (int step = 0; step < f->F.max_steps; ++step) {
    const bool fz = fused && step == 0;
    unsigned long long* srow =
        step_rows && (step_stride == 0 || step < DDF_STAGE_STEPS) ? step_rows + step * step_stride : nullptr;
    if (fz) {
      int rc = compact_flags(f, ms.alive, nullptr, n, 1, list, sm.seg, sm.count, fwd_acc, st, want, 1, sm.stats + 3,
                             srow);
      if (rc) return rc;
      if ((rc = stage_log(f, lg, list, sm.count, 3, bounce, step, st))) return rc;
      TraceGradOp op = *fused;
      op.list = list; op.count = sm.count; op.n = n; op.seg = nullptr;
      op.st = ms; op.delta = f->F.delta; op.thresh = f->F.thresh; op.step = f->F.step;
      if ((rc = run_fused(f, op, n, st))) return rc;
    }
    int rc = compact_flags(f, ms.alive, nullptr, n, 1, list, sm.seg, sm.count, fwd_acc, st, fz ? want : nullptr, 0,
                           srow);
    if (rc) return rc;
    if ((rc = stage_log(f, lg, list, sm.count, bounce < 0 ? 0 : 2, bounce, step, st))) return rc;
    TraceStepOp op{};
    op.list = list; op.count = sm.count; op.n = n; op.seg = nullptr;
    op.st = ms; op.delta = f->F.delta; op.thresh = f->F.thresh; op.step = f->F.step;
    rc = run_mlp(f, f->F, op, n, false, st);
    if (rc) return rc;
  }
  return DDF_OK;
}

void build_stream(const uint64_t st[2], const uint64_t inc[2], PcgStream* out) {
  typedef unsigned __int128 U;
  const U mult = ((U)0x2360ED051FC65DA4ull << 64) | (U)0x4385DF649FCCF645ull;
  U cm = mult, cp = ((U)inc[1] << 64) | inc[0];
  out->state = u128{st[0], st[1]};
  for (int b = 0; b < 64; ++b) {
    out->mult[b] = u128{(uint64_t)cm, (uint64_t)(cm >> 64)};
    out->plus[b] = u128{(uint64_t)cp, (uint64_t)(cp >> 64)};
    cp = (cm + 1) * cp;
    cm = cm * cm;
  }
}

int ensure_small(ddf_field_s* f) {
  CUDA_TRY(f->small.ensure(4096));
  return DDF_OK;
}

bool has_geometry(const ddf_field_s* f) { return f && (f->F.n_obj > 0 || f->F.is_mesh); }

// ---------------------------------------------------------------- mesh BVH (mesh.py:94-166)
// Median split on the longest box axis, <= 4 triangles per leaf, built once
// on the host.  The partition (std::nth_element) may order equal centroids
// differently from numpy's argpartition; hits do not depend on the tree.
int build_mesh(ddf_field_s* f, const double* V, int64_t nv, const int32_t* Fc, int64_t nf) {
  using mesh::Node;
  using mesh::Tri;
  const int LEAF = 4;
  std::vector<double> tmin(3 * nf), tmax(3 * nf), cent(3 * nf);
  for (int64_t i = 0; i < nf; ++i) {
    for (int k = 0; k < 3; ++k) {
      const double a = V[3 * Fc[3 * i] + k], b = V[3 * Fc[3 * i + 1] + k], c = V[3 * Fc[3 * i + 2] + k];
      tmin[3 * i + k] = std::min(std::min(a, b), c);
      tmax[3 * i + k] = std::max(std::max(a, b), c);
      cent[3 * i + k] = ((a + b) + c) / 3.0;
    }
  }
  std::vector<int> prim(nf);
  for (int64_t i = 0; i < nf; ++i) prim[i] = (int)i;
  std::vector<Node> nodes;
  nodes.reserve(2 * (size_t)(nf / LEAF + 1));
  struct Job { int node, lo, hi; };
  std::vector<Job> stack;
  nodes.push_back(Node{});
  stack.push_back({0, 0, (int)nf});
  while (!stack.empty()) {
    const Job j = stack.back();
    stack.pop_back();
    Node nd{};
    for (int k = 0; k < 3; ++k) { nd.lo[k] = INFINITY; nd.hi[k] = -INFINITY; }
    for (int i = j.lo; i < j.hi; ++i)
      for (int k = 0; k < 3; ++k) {
        nd.lo[k] = std::min(nd.lo[k], tmin[3 * prim[i] + k]);
        nd.hi[k] = std::max(nd.hi[k], tmax[3 * prim[i] + k]);
      }
    if (j.hi - j.lo <= LEAF) {
      nd.left = nd.right = -1;
      nd.start = j.lo;
      nd.count = j.hi - j.lo;
      nodes[j.node] = nd;
      continue;
    }
    int axis = 0;
    for (int k = 1; k < 3; ++k)
      if (nd.hi[k] - nd.lo[k] > nd.hi[axis] - nd.lo[axis]) axis = k;
    const int mid = (j.lo + j.hi) / 2;
    std::nth_element(prim.begin() + j.lo, prim.begin() + mid, prim.begin() + j.hi,
                     [&](int a, int b) { return cent[3 * a + axis] < cent[3 * b + axis]; });
    const int lc = (int)nodes.size();
    nodes.push_back(Node{});
    const int rc = (int)nodes.size();
    nodes.push_back(Node{});
    nd.left = lc;
    nd.right = rc;
    nd.start = nd.count = 0;
    nodes[j.node] = nd;
    stack.push_back({rc, mid, j.hi});
    stack.push_back({lc, j.lo, mid});
  }
  std::vector<Tri> tris(nf);
  std::vector<int> tof(nf);
  for (int64_t k = 0; k < nf; ++k) {
    const int i = prim[k];
    Tri T{};
    for (int c = 0; c < 3; ++c) {
      T.a[c] = V[3 * Fc[3 * i] + c];
      T.b[c] = V[3 * Fc[3 * i + 1] + c];
      T.c[c] = V[3 * Fc[3 * i + 2] + c];
    }
    T.face = i;
    tris[k] = T;
    tof[i] = (int)k;
  }
  (void)nv;
  CUDA_TRY(f->mesh_nodes.ensure(sizeof(Node) * nodes.size()));
  CUDA_TRY(f->mesh_tris.ensure(sizeof(Tri) * tris.size()));
  CUDA_TRY(f->mesh_tof.ensure(sizeof(int) * tof.size()));
  CUDA_TRY(cudaMemcpy(f->mesh_nodes.p, nodes.data(), sizeof(Node) * nodes.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(f->mesh_tris.p, tris.data(), sizeof(Tri) * tris.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(f->mesh_tof.p, tof.data(), sizeof(int) * tof.size(), cudaMemcpyHostToDevice));
  f->M.nodes = f->mesh_nodes.as<Node>();
  f->M.tris = f->mesh_tris.as<Tri>();
  f->M.tri_of_face = f->mesh_tof.as<int>();
  f->M.n_faces = (int)nf;
  return DDF_OK;
}

// ---------------------------------------------------------------- UDF (field.py:418-488)
__global__ void twice_kernel(const int* c, int* c2) { *c2 = 2 * *c; }

// field.py:115-141 sphere_directions on the host in float64 (setup, not hot)
std::vector<double> sphere_directions(int n) {
  auto vdc = [](long long i, int base) {
    double out = 0.0, scale = 1.0 / base;
    while (i > 0) {
      out += scale * (double)(i % base);
      i /= base;
      scale /= base;
    }
    return out;
  };
  const double two_pi = 2.0 * 3.141592653589793;
  std::vector<double> d(3 * (size_t)n);
  for (int k = 0; k < n; ++k) {
    const double z = 1.0 - 2.0 * vdc(k + 1, 2);
    const double phi = two_pi * vdc(k + 1, 3);
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    d[3 * k] = r * std::cos(phi);
    d[3 * k + 1] = r * std::sin(phi);
    d[3 * k + 2] = z;
  }
  return d;
}

constexpr int64_t UDF_CHUNK_ROWS = 1ll << 25;   // scan rows per chunk: 256 MB of f64 values
constexpr int64_t UDF_POLISH_PTS = 1ll << 22;   // points per polish pass: 4M x 76 B of state

int udf_run(ddf_field_s* f, const double* pts, int64_t n, int n_dirs, bool polish, double* out, cudaStream_t st) {
  if (n_dirs < 1) return fail(DDF_EUSAGE, "need at least one direction");
  if (n_dirs > (1 << 24)) return fail(DDF_EUSAGE, "n_dirs too large");
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad point count");
  if (n == 0) return DDF_OK;
  if (f->udf_ndirs != n_dirs) {
    const std::vector<double> d = sphere_directions(n_dirs);
    CUDA_TRY(f->udf_dirs.ensure(sizeof(double) * 5 * n_dirs));     // dirs (n,3) + encoded angles (n,2)
    CUDA_TRY(cudaMemcpy(f->udf_dirs.p, d.data(), sizeof(double) * d.size(), cudaMemcpyHostToDevice));
    udf::dir_u34_kernel<<<(n_dirs + 127) / 128, 128>>>(f->udf_dirs.as<double>(), n_dirs,
                                                        f->udf_dirs.as<double>() + 3 * n_dirs);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    f->udf_ndirs = n_dirs;
  }
  const double* dirs = f->udf_dirs.as<double>();
  const double* dir_u34 = dirs + 3 * n_dirs;
  const int64_t pc = std::min<int64_t>(n, UDF_POLISH_PTS);                       // polish pass
  const int64_t sc = std::max<int64_t>(1, std::min<int64_t>(pc, UDF_CHUNK_ROWS / n_dirs));   // scan chunk
  CUDA_TRY(f->udf_vals.ensure(sizeof(double) * sc * n_dirs));
  CUDA_TRY(f->udf_arg.ensure(sizeof(int) * pc));
  CUDA_TRY(f->udf_found.ensure(pc));
  CUDA_TRY(f->udf_list.ensure(sizeof(int) * pc));
  CUDA_TRY(f->udf_seg.ensure(sizeof(int) * 4));
  if (polish) CUDA_TRY(f->udf_state.ensure(sizeof(double) * 9 * pc));
  const double golden = (std::sqrt(5.0) - 1.0) / 2.0;        // field.py:406
  const double half = 3.0 / std::sqrt((double)n_dirs);        // field.py:454
  for (int64_t q0 = 0; q0 < n; q0 += pc) {
    const int nq = (int)std::min<int64_t>(pc, n - q0);
    const double* P = pts + 3 * q0;
    double* best = out + q0;
    // stage 1: direction scan + first argmin, chunked by the value buffer
    for (int64_t p0 = 0; p0 < nq; p0 += sc) {
      const int np_ = (int)std::min<int64_t>(sc, nq - p0);
      udf::ScanOp op{};
      op.list = nullptr; op.count = nullptr; op.n = np_ * n_dirs; op.seg = nullptr;
      op.pts = P + 3 * p0; op.u34 = dir_u34; op.n_dirs = n_dirs; op.vals = f->udf_vals.as<double>();
      op.delta = f->F.delta; op.thresh = f->F.thresh;
      if (int rc = run_mlp(f, f->F, op, op.n, false, st)) return rc;
      f->prof.launches += 1;
      udf::reduce_kernel<<<(np_ + 7) / 8, 256, 0, st>>>(op.vals, np_, n_dirs, best + p0,
                                                         f->udf_arg.as<int>() + p0, f->udf_found.as<uint8_t>() + p0);
      CUDA_TRY(cudaGetLastError());
    }
    if (!polish) continue;
    // stage 2: golden-section polish of every found point of this pass
    int* cnt = f->udf_seg.as<int>() + 2;
    if (int rc = compact_flags(f, f->udf_found.as<uint8_t>(), nullptr, nq, 1, f->udf_list.as<int>(),
                               f->udf_seg.as<int>(), cnt, nullptr, st))
      return rc;
    int* cnt2 = cnt + 1;
    twice_kernel<<<1, 1, 0, st>>>(cnt, cnt2);
    double* S = f->udf_state.as<double>();
    udf::Polish G{f->udf_list.as<int>(), S, S + 2 * pc, S + 3 * pc, S + 4 * pc, S + 5 * pc, S + 6 * pc,
                  S + 7 * pc, S + 8 * pc};
    const int nb = (nq + 255) / 256;
    f->prof.launches += 3;
    udf::polish_init<<<nb, 256, 0, st>>>(G, f->udf_arg.as<int>(), best, dirs, nq, cnt);
    udf::ProbeOp pr{};
    pr.list = nullptr; pr.count = cnt2; pr.n = 2 * nq; pr.seg = nullptr;
    pr.pts = P; pr.P = G; pr.delta = f->F.delta; pr.thresh = f->F.thresh;
    for (int round = 0; round < 2; ++round) {
      for (int axis = 1; axis >= 0; --axis) {                  // field.py:457 (polar, then azimuth)
        pr.axis = axis;
        udf::gs_begin<<<nb, 256, 0, st>>>(G, axis, half, golden, nq, cnt);
        if (int rc = run_mlp(f, f->F, pr, 2 * nq, false, st)) return rc;
        for (int it = 0; it < 12; ++it) {                       // field.py:476
          udf::gs_step<<<nb, 256, 0, st>>>(G, golden, nq, cnt);
          if (int rc = run_mlp(f, f->F, pr, 2 * nq, false, st)) return rc;
        }
        udf::gs_end<<<nb, 256, 0, st>>>(G, axis, nq, cnt);
        f->prof.launches += 14;
      }
    }
    udf::polish_scatter<<<nb, 256, 0, st>>>(G, best, nq, cnt);
    CUDA_TRY(cudaGetLastError());
  }
  return DDF_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* ddf_last_error(void) { return g_err.c_str(); }

int ddf_field_create(double delta, const double bounds[6], int32_t precision, int32_t device, ddf_field_t* out) {
  if (!out) return fail(DDF_EUSAGE, "null output handle");
  if (!(delta > 0.0)) return fail(DDF_EUSAGE, "delta must be positive");
  if (precision != DDF_PREC_FP32 && precision != DDF_PREC_BF16 && precision != DDF_PREC_FP32_SIMT)
    return fail(DDF_EUSAGE, "unknown precision");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(DDF_ECUDA, "no CUDA device: the B200 DDF path has no CPU fallback");
  if (device < 0 || device >= ndev) return fail(DDF_EUSAGE, "bad device index");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(DDF_ECUDA, "libddf_b200 is built for sm_100a (B200) only");
  auto* f = new ddf_field_s();
  f->device = device;
  f->sm_count = prop.multiProcessorCount;
  FieldDev& F = f->F;
  F.n_obj = 0;
  F.precision = precision;
  F.delta = delta;
  for (int k = 0; k < 3; ++k) { F.lo[k] = bounds[k]; F.hi[k] = bounds[3 + k]; }
  F.step = 0.9 * delta;
  F.thresh = DDF_HIT_FRACTION * delta;
  F.backoff = 0.5 * delta;
  const double dx = bounds[3] - bounds[0], dy = bounds[4] - bounds[1], dz = bounds[5] - bounds[2];
  const double diag = std::sqrt((dx * dx + dy * dy) + dz * dz);
  F.max_steps = (int)std::ceil(diag / F.step) + 4;
  F.composite = false;
  if (cudaMalloc(&f->F_dev, sizeof(FieldDev)) != cudaSuccess) {
    delete f;
    return fail(DDF_ECUDA, "cudaMalloc failed");
  }
  *out = f;
  return DDF_OK;
}

int ddf_field_add_network(ddf_field_t f, const int32_t* widths, int32_t n_widths, const double* weights,
                          const double* biases, int32_t encoding, const double center[3], double scale,
                          double albedo) {
  if (!f || !widths || !weights || !biases) return fail(DDF_EUSAGE, "null argument");
  if (f->F.n_obj >= DDF_MAX_OBJECTS) return fail(DDF_EUSAGE, "too many networks in one field");
  const int L = n_widths - 1;
  if (L < 1 || L > DDF_MAX_LAYERS) return fail(DDF_EUSAGE, "unsupported layer count");
  if (widths[L] != 1) return fail(DDF_EDATA, "network head must have width 1");
  for (int l = 0; l < n_widths; ++l)
    if (widths[l] < 1) return fail(DDF_EDATA, "bad layer width");
  if (encoding == DDF_ENC_RAW5 && widths[0] != 5) encoding = 2;   // raw-input ops only (ddf_mlp_*)
  if (encoding == DDF_ENC_PE6 && widths[0] != 65) return fail(DDF_EDATA, "PE encoding needs 65 inputs");
  if (!(scale > 0.0)) return fail(DDF_EUSAGE, "scale must be positive");
  CUDA_TRY(cudaSetDevice(f->device));
  NetDev& N = f->F.net[f->F.n_obj];
  N = NetDev{};
  N.n_layers = L;
  N.encoding = encoding;
  for (int k = 0; k < 3; ++k) N.center[k] = center ? center[k] : 0.0;
  N.scale = scale;
  N.inv_scale = 1.0 / scale;
  N.albedo = albedo;
  std::vector<int> wp(L + 1);
  for (int l = 0; l < L; ++l) wp[l] = pad16(widths[l]);
  wp[L] = 1;
  for (int l = 0; l <= L; ++l) N.widths[l] = wp[l];
  N.max_width = *std::max_element(wp.begin(), wp.end());
  size_t woff = 0, boff = 0;
  for (int l = 0; l < L; ++l) {
    const int in = widths[l], out = widths[l + 1], pin = wp[l], pout = wp[l + 1];
    std::vector<float> w((size_t)pout * pin, 0.f), wt((size_t)pin * pout, 0.f), b(pout, 0.f);
    for (int o = 0; o < out; ++o) {
      for (int i = 0; i < in; ++i) {
        const float v = (float)weights[woff + (size_t)o * in + i];
        w[(size_t)o * pin + i] = v;
        wt[(size_t)i * pout + o] = v;
      }
      b[o] = (float)biases[boff + o];
    }
    woff += (size_t)out * in;
    boff += out;
    float *dw, *dwt, *db;
    CUDA_TRY(cudaMalloc(&dw, w.size() * 4));
    CUDA_TRY(cudaMalloc(&dwt, wt.size() * 4));
    CUDA_TRY(cudaMalloc(&db, std::max<size_t>(16, b.size() * 4)));
    CUDA_TRY(cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dwt, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
    f->weights.push_back(dw);
    f->weights.push_back(dwt);
    f->weights.push_back(db);
    N.w[l] = dw;
    N.wt[l] = dwt;
    N.b[l] = db;
  }
  // bf16 UMMA weight images (built for every net; used when precision == BF16)
  // A linear model (no hidden layer, a legal reference MlpModel) has no GEMM
  // for the tensor cores: it runs on the SIMT kernel in both precisions.
  umma::NetImage img{};
  img.in_width = widths[0];
  if (L >= 2) {
    int rc = umma::build_image(widths, n_widths, weights, biases, &img, &g_err);
    if (rc) return rc;
  }
  f->images.push_back(img);
  N.wimg_fwd = img.dev;
  N.wimg_bwd = img.dev;
  // 3xTF32 images (fp32 mode on the tensor cores) when the widths fit the engine
  umma::NetImage img3{};
  img3.in_width = widths[0];
  if (x3::supports(widths, n_widths)) {
    int rc = x3::build_image(widths, n_widths, weights, biases, &img3, &g_err);
    if (rc) return rc;
  }
  f->images_x3.push_back(img3);
  N.wimg_x3 = img3.dev;
  f->F.n_obj += 1;
  f->gen += 1;
  // composite as soon as there is more than one object or a transform
  bool comp = f->F.n_obj > 1;
  for (int j = 0; j < f->F.n_obj; ++j) {
    const NetDev& n = f->F.net[j];
    if (n.scale != 1.0 || n.center[0] != 0.0 || n.center[1] != 0.0 || n.center[2] != 0.0) comp = true;
  }
  f->F.composite = comp;
  CUDA_TRY(cudaMemcpy(f->F_dev, &f->F, sizeof(FieldDev), cudaMemcpyHostToDevice));
  return DDF_OK;
}

int ddf_field_set_precision(ddf_field_t f, int32_t precision) {
  if (!f) return fail(DDF_EUSAGE, "null field");
  if (precision != DDF_PREC_FP32 && precision != DDF_PREC_BF16 && precision != DDF_PREC_FP32_SIMT)
    return fail(DDF_EUSAGE, "unknown precision");
  f->F.precision = precision;
  f->gen += 1;
  CUDA_TRY(cudaSetDevice(f->device));
  CUDA_TRY(cudaMemcpy(f->F_dev, &f->F, sizeof(FieldDev), cudaMemcpyHostToDevice));
  return DDF_OK;
}

int ddf_field_destroy(ddf_field_t f) {
  if (!f) return DDF_OK;
  cudaSetDevice(f->device);
  for (void* p : f->weights) cudaFree(p);
  for (auto& im : f->images) umma::free_image(&im);
  for (auto& im : f->images_x3) umma::free_image(&im);
  Buf* bufs[] = {&f->t_acc, &f->t_exit, &f->alive, &f->list, &f->list2, &f->blocks, &f->small, &f->ones, &f->op_state,
                 &f->st_o, &f->st_d, &f->st_tacc, &f->st_texit, &f->st_t, &f->st_thr, &f->st_rad,
                 &f->st_hit, &f->st_march, &f->st_alive, &f->st_obj, &f->pix, &f->rng, &f->umma_masks, &f->st_u34, &f->st_g3, &f->st_gdone, &f->st_want,
                 &f->udf_dirs, &f->udf_vals, &f->udf_pts, &f->udf_best, &f->udf_arg, &f->udf_found, &f->udf_list,
                 &f->udf_seg, &f->udf_state, &f->mesh_nodes, &f->mesh_tris, &f->mesh_tof};
  for (Buf* b : bufs) b->release();
  if (f->F_dev) cudaFree(f->F_dev);
  if (f->graph_exec) cudaGraphExecDestroy(f->graph_exec);
  if (f->cap_stream) cudaStreamDestroy(f->cap_stream);
  delete f;
  return DDF_OK;
}

static int check_net(ddf_field_t f, int net) {
  if (!f) return fail(DDF_EUSAGE, "null field");
  if (net < 0 || net >= f->F.n_obj) return fail(DDF_EUSAGE, "bad network index");
  return DDF_OK;
}

static FieldDev single_net(const FieldDev& F, int net) {
  FieldDev G = F;
  G.n_obj = 1;
  G.composite = false;
  G.net[0] = F.net[net];
  return G;
}

int ddf_mlp_forward(ddf_field_t f, int32_t net, const double* x, int64_t n, double* out, void* stream) {
  if (int rc = check_net(f, net)) return rc;
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad row count");
  if (n == 0) return DDF_OK;
  CUDA_TRY(cudaSetDevice(f->device));
  RawForwardOp op{};
  op.list = nullptr; op.count = nullptr; op.n = (int)n; op.seg = nullptr;
  op.x = x; op.width = f->images[net].in_width; op.out = out;   // unpadded row stride
  return run_mlp(f, single_net(f->F, net), op, (int)n, false, (cudaStream_t)stream);
}

int ddf_mlp_input_grad(ddf_field_t f, int32_t net, const double* x, int64_t n, double* out, void* stream) {
  if (int rc = check_net(f, net)) return rc;
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad row count");
  if (n == 0) return DDF_OK;
  CUDA_TRY(cudaSetDevice(f->device));
  RawGradOp op{};
  op.list = nullptr; op.count = nullptr; op.n = (int)n; op.seg = nullptr;
  op.x = x; op.width = f->images[net].in_width; op.out = out;
  return run_mlp(f, single_net(f->F, net), op, (int)n, true, (cudaStream_t)stream);
}

int ddf_query(ddf_field_t f, const double* pos, const double* dirs, int64_t n, double* t, uint8_t* hit,
              double* pred, int32_t* obj, void* stream) {
  if (!has_geometry(f)) return fail(DDF_EUSAGE, "field has no network");
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad row count");
  if (n == 0) return DDF_OK;
  CUDA_TRY(cudaSetDevice(f->device));
  if (f->F.is_mesh) {
    mesh::query_kernel<<<(int)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(f->M, pos, dirs, (int)n, t, hit,
                                                                               pred, obj);
    CUDA_TRY(cudaGetLastError());
    return DDF_OK;
  }
  QueryOp op{};
  op.list = nullptr; op.count = nullptr; op.n = (int)n; op.seg = nullptr;
  op.pos = pos; op.dirs = dirs; op.t = t; op.hit = hit; op.pred_out = pred; op.obj_out = obj;
  op.delta = f->F.delta; op.thresh = f->F.thresh;
  return run_mlp(f, f->F, op, (int)n, false, (cudaStream_t)stream);
}

int ddf_trace(ddf_field_t f, const double* origins, const double* dirs, int64_t n, double* t, uint8_t* hit,
              int32_t* obj, void* stream) {
  if (!has_geometry(f)) return fail(DDF_EUSAGE, "field has no network");
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad row count");
  if (n == 0) return DDF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(f->device));
  if (f->F.is_mesh) {   // trace_batch = query_batch for mesh fields (field.py:170)
    mesh::query_kernel<<<(int)((n + 127) / 128), 128, 0, st>>>(f->M, origins, dirs, (int)n, t, hit, nullptr, obj);
    CUDA_TRY(cudaGetLastError());
    return DDF_OK;
  }
  if (int rc = ensure_small(f)) return rc;
  CUDA_TRY(f->t_acc.ensure(sizeof(double) * n));
  CUDA_TRY(f->t_exit.ensure(sizeof(double) * n));
  CUDA_TRY(f->alive.ensure(n));
  CUDA_TRY(f->list.ensure(sizeof(int) * n));
  CUDA_TRY(f->st_obj.ensure(sizeof(int) * n));
  MarchState ms{};
  ms.o = origins; ms.d = dirs;
  ms.t_acc = f->t_acc.as<double>(); ms.t_exit = f->t_exit.as<double>();
  ms.alive = f->alive.as<uint8_t>(); ms.t_out = t; ms.hit = hit;
  ms.obj = obj ? obj : f->st_obj.as<int>();
  trace_init_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(f->F, ms, (int)n);
  CUDA_TRY(cudaGetLastError());
  return march(f, ms, (int)n, f->list.as<int>(), nullptr, st);
}

int ddf_normal(ddf_field_t f, const double* origins, const double* dirs, const double* t_hit, const int32_t* obj,
               int64_t n, double* normals, uint8_t* valid, void* stream) {
  if (!has_geometry(f)) return fail(DDF_EUSAGE, "field has no network");
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad row count");
  if (n == 0) return DDF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(f->device));
  if (f->F.is_mesh) {   // re-intersects (field.py:174-176); t_hit and obj are not used
    mesh::normal_kernel<<<(int)((n + 127) / 128), 128, 0, st>>>(f->M, origins, dirs, (int)n, normals, valid);
    CUDA_TRY(cudaGetLastError());
    return DDF_OK;
  }
  if (int rc = ensure_small(f)) return rc;
  NormalOp op{};
  op.o = origins; op.d = dirs; op.t_hit = t_hit; op.backoff = f->F.backoff; op.normals = normals; op.valid = valid;
  op.n = (int)n; op.count = nullptr; op.list = nullptr; op.seg = nullptr;
  if (f->F.n_obj > 1) {
    if (!obj) return fail(DDF_EUSAGE, "composite fields need the hit object ids for normals");
    CUDA_TRY(f->ones.ensure(n));
    CUDA_TRY(cudaMemsetAsync(f->ones.p, 1, n, st));
    CUDA_TRY(f->list.ensure(sizeof(int) * n));
    Small sm = small_of(f);
    if (int rc = compact_flags(f, f->ones.as<uint8_t>(), obj, (int)n, f->F.n_obj, f->list.as<int>(), sm.seg,
                               sm.count, nullptr, st))
      return rc;
    op.list = f->list.as<int>(); op.count = sm.count; op.seg = sm.seg;
  }
  return run_mlp(f, f->F, op, (int)n, true, st);
}

int ddf_render_path(ddf_field_t f, const ddf_camera_t* cam, const ddf_path_config_t* cfg, double* accum,
                    ddf_render_stats_t* stats, void* stream) {
  if (!has_geometry(f)) return fail(DDF_EUSAGE, "field has no network");
  if (!cam || !cfg || !accum) return fail(DDF_EUSAGE, "null argument");
  if (cfg->bounces < 1) return fail(DDF_EUSAGE, "path mode needs bounces >= 1");   // render.py:207-208
  if (cfg->spp < 1) return fail(DDF_EUSAGE, "spp must be >= 1");                 // render.py:119-120
  if (cam->width < 1 || cam->height < 1) return fail(DDF_EUSAGE, "film dimensions must be >= 1");
  const int64_t n_pix = (int64_t)cam->width * cam->height;
  if (n_pix > (1ll << 30)) return fail(DDF_EUSAGE, "film too large");
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world || cfg->tile < 0)
    return fail(DDF_EUSAGE, "bad tile sharding");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(f->device));
  if (int rc = ensure_small(f)) return rc;
  Small sm = small_of(f);
  f->prof.reset(cfg->profile != 0);
  size_t t_begin = f->prof.on ? f->prof.rec(st) : 0;

  // owned pixels, ascending global index (cached per film/sharding/owner table)
  const int key[6] = {cam->width, cam->height, cfg->tile, cfg->rank, cfg->world, 1};
  const int T = cfg->tile;
  const int ntx = T > 0 ? (cam->width + T - 1) / T : 1;
  const int nty = T > 0 ? (cam->height + T - 1) / T : 1;
  std::vector<int32_t> owner;
  if (cfg->tile_owner && T > 0) {
    owner.assign(cfg->tile_owner, cfg->tile_owner + (size_t)ntx * nty);
    for (int32_t r : owner)
      if (r < 0 || r >= cfg->world) return fail(DDF_EUSAGE, "tile_owner entry out of [0, world)");
  }
  if (std::memcmp(key, f->pix_key, sizeof(key)) != 0 || owner != f->pix_owner) {
    std::vector<int> own;
    own.reserve(n_pix / cfg->world + 1);
    if (T > 0) {
      // row-major walk one tile-row segment at a time: ascending global ids,
      // O(H * ntx) ownership tests (the pilot calls this once per tile)
      for (int py = 0; py < cam->height; ++py)
        for (int tx = 0; tx < ntx; ++tx) {
          const int tile_id = (py / T) * ntx + tx;
          if ((owner.empty() ? tile_id % cfg->world : owner[tile_id]) != cfg->rank) continue;
          const int x1 = std::min(cam->width, (tx + 1) * T);
          for (int px = tx * T; px < x1; ++px) own.push_back(py * cam->width + px);
        }
    } else {
      for (int64_t i = 0; i < n_pix; ++i)
        if (cfg->world == 1 || (i % cfg->world) == cfg->rank) own.push_back((int)i);
    }
    CUDA_TRY(f->pix.ensure(sizeof(int) * std::max<size_t>(1, own.size())));
    if (!own.empty())
      CUDA_TRY(cudaMemcpy(f->pix.p, own.data(), sizeof(int) * own.size(), cudaMemcpyHostToDevice));
    std::memcpy(f->pix_key, key, sizeof(key));
    f->pix_owner = owner;
    f->pix_n = (int)own.size();
  }
  const int n_own = f->pix_n;
  CUDA_TRY(cudaMemsetAsync(f->small.p, 0, 4096, st));
  if (n_own == 0) {
    CUDA_TRY(cudaMemsetAsync(accum, 0, sizeof(double) * n_pix, st));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    f->prof.reset(false);
    return DDF_OK;
  }

  // RNG jump tables
  PcgStream hs[2];
  build_stream(cfg->rng_state, cfg->rng_inc, &hs[0]);
  build_stream(cfg->rr_state, cfg->rr_inc, &hs[1]);
  CUDA_TRY(f->rng.ensure(sizeof(hs)));
  CUDA_TRY(cudaMemcpyAsync(f->rng.p, hs, sizeof(hs), cudaMemcpyHostToDevice, st));

  // wave sizing
  int64_t maxp = cfg->max_wave_paths > 0 ? cfg->max_wave_paths : (int64_t)8 << 20;
  int ns = (int)std::max<int64_t>(1, std::min<int64_t>(cfg->spp, maxp / n_own));
  const int64_t P64 = (int64_t)ns * n_own;
  if (P64 > (1ll << 30)) return fail(DDF_EUSAGE, "wave too large");
  const int P = (int)P64;
  CUDA_TRY(f->st_o.ensure(sizeof(double) * 3 * P));
  CUDA_TRY(f->st_d.ensure(sizeof(double) * 3 * P));
  CUDA_TRY(f->st_tacc.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_texit.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_t.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_thr.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_rad.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_hit.ensure(P));
  CUDA_TRY(f->st_march.ensure(P));
  CUDA_TRY(f->st_alive.ensure(P));
  CUDA_TRY(f->st_obj.ensure(sizeof(int) * P));
  CUDA_TRY(f->st_u34.ensure(sizeof(double) * 2 * P));
  CUDA_TRY(f->st_g3.ensure(sizeof(double) * 3 * P));
  CUDA_TRY(f->st_gdone.ensure(P));
  CUDA_TRY(f->st_want.ensure(P));
  CUDA_TRY(f->list.ensure(sizeof(int) * P));
  CUDA_TRY(f->list2.ensure(sizeof(int) * P));
  CUDA_TRY(f->film.ensure(sizeof(double) * n_pix));
  double* film = f->film.as<double>();
  CUDA_TRY(cudaMemsetAsync(film, 0, sizeof(double) * n_pix, st));

  PathState S{};
  S.o = f->st_o.as<double>(); S.d = f->st_d.as<double>();
  S.t_acc = f->st_tacc.as<double>(); S.t_exit = f->st_texit.as<double>(); S.t = f->st_t.as<double>();
  S.thr = f->st_thr.as<double>(); S.rad = f->st_rad.as<double>();
  S.hit = f->st_hit.as<uint8_t>(); S.march = f->st_march.as<uint8_t>(); S.alive = f->st_alive.as<uint8_t>();
  S.obj = f->st_obj.as<int>();
  S.u34 = f->st_u34.as<double>();
  S.g3 = f->st_g3.as<double>();
  S.gdone = f->st_gdone.as<uint8_t>();
  S.want = f->st_want.as<uint8_t>();
  const bool fuse = !cfg->no_fuse && fusion_ok(f);
  TraceGradOp tg{};
  tg.backoff = f->F.backoff; tg.g3 = S.g3; tg.gdone = S.gdone;
  MarchState ms{};
  ms.o = S.o; ms.d = S.d; ms.t_acc = S.t_acc; ms.t_exit = S.t_exit; ms.alive = S.march;
  ms.t_out = S.t; ms.hit = S.hit; ms.obj = S.obj; ms.u34 = S.u34;

  CamDev C{};
  for (int k = 0; k < 3; ++k) {
    C.pos[k] = cam->position[k]; C.fwd[k] = cam->forward[k]; C.right[k] = cam->right[k]; C.up[k] = cam->up_ortho[k];
  }
  C.tan_half = cam->tan_half; C.aspect = cam->aspect; C.W = cam->width; C.H = cam->height;

  WaveDev w{};
  w.spp = cfg->spp; w.bounces = cfg->bounces; w.albedo = cfg->albedo; w.env = cfg->env_radiance;
  w.rr_start = cfg->rr_start; w.n_pix = n_pix; w.pix = f->pix.as<int>(); w.n_own = n_own;
  w.rng = f->rng.as<PcgStream>(); w.rr = f->rng.as<PcgStream>() + 1;
  w.err = sm.err; w.degenerate = sm.stats + 2;

  // stage log (debug): the header is cleared once per render
  const bool lg_on = cfg->stage_log != nullptr;
  if (lg_on && cfg->stage_log_cap < 2) return fail(DDF_EUSAGE, "stage_log needs at least 2 words");
  StageLog lg;
  lg.log = cfg->stage_log; lg.cap = cfg->stage_log_cap; lg.n_own = n_own;
  if (lg_on) CUDA_TRY(cudaMemsetAsync(lg.log, 0, 2 * sizeof(int), st));

  int waves = 0;
  // the wave loop: stream-ordered launches only (no host syncs, no
  // allocations once the buffers have grown), so it can be captured
  auto run_waves = [&](cudaStream_t ss) -> int {
    waves = 0;
    for (int s0 = 0; s0 < cfg->spp; s0 += ns) {
      w.s0 = s0;
      lg.s0 = s0;
      w.ns = std::min(ns, cfg->spp - s0);
      const int Pw = w.ns * n_own;
      const int g = (Pw + 255) / 256;
      {
        ProfScope ps(f->prof, Prof::CAMERA, ss);
        camera_kernel<<<g, 256, 0, ss>>>(f->F, C, w, S, Pw);
        f->prof.launches += 1;
      }
      CUDA_TRY(cudaGetLastError());
      if (f->F.is_mesh) {
        ProfScope ps(f->prof, Prof::FWD, ss);
        mesh::trace_paths_kernel<<<g, 256, 0, ss>>>(f->M, S, nullptr, nullptr, Pw);
        f->prof.launches += 1;
        f->prof.fwd_launches += 1;
      } else if (int rc = march(f, ms, Pw, f->list2.as<int>(), sm.stats + 0, ss, nullptr, nullptr,
                                sm.primary_rows(), 1, lg_on ? &lg : nullptr, -1)) {
        return rc;
      }
      {
        ProfScope ps(f->prof, Prof::AFTER, ss);
        after_primary_kernel<<<g, 256, 0, ss>>>(w, S, Pw);
        f->prof.launches += 1;
      }
      for (int b = 0; b < cfg->bounces; ++b) {
        if (cfg->rr_start >= 0 && b >= cfg->rr_start) {
          ProfScope ps(f->prof, Prof::ROULETTE, ss);
          roulette_kernel<<<g, 256, 0, ss>>>(w, S, Pw, b);
          f->prof.launches += 1;
        }
        int rc = compact_flags(f, S.alive, f->F.n_obj > 1 ? S.obj : nullptr, Pw, f->F.n_obj, f->list.as<int>(),
                               sm.seg, sm.count2, sm.stats + 1, ss, nullptr, 0,
                               b < DDF_STAGE_BOUNCES ? sm.alive_rows() + b : nullptr);
        if (rc) return rc;
        if ((rc = stage_log(f, lg_on ? &lg : nullptr, f->list.as<int>(), sm.count2, 1, b, 0, ss))) return rc;
        if (f->F.is_mesh) {
          ProfScope ps(f->prof, Prof::GRAD, ss);
          mesh::face_normal_kernel<<<std::min(g, f->sm_count * 8), 256, 0, ss>>>(f->M, S, f->list.as<int>(), sm.count2);
          f->prof.launches += 1;
          f->prof.grad_launches += 1;
        } else if (fuse) {
          // rows whose normal gradient the fused trace step already produced are left out
          if ((rc = compact_flags(f, S.alive, nullptr, Pw, 1, f->list2.as<int>(), sm.seg, sm.count, sm.stats + 4, ss,
                                  S.gdone, 0)))
            return rc;
          GradOutOp op{};
          op.list = f->list2.as<int>(); op.count = sm.count; op.n = Pw; op.seg = nullptr;
          op.S = S; op.backoff = f->F.backoff;
          if ((rc = run_mlp(f, f->F, op, Pw, true, ss))) return rc;
        } else {
          GradOutOp op{};
          op.list = f->list.as<int>(); op.count = sm.count2; op.n = Pw;
          op.seg = f->F.n_obj > 1 ? sm.seg : nullptr;
          op.S = S; op.backoff = f->F.backoff;
          if ((rc = run_mlp(f, f->F, op, Pw, true, ss))) return rc;
        }
        {
          ProfScope ps(f->prof, Prof::BOUNCE, ss);
          bounce_kernel<<<std::min(g, f->sm_count * 8), 256, 0, ss>>>(f->F_dev, w, S, f->list.as<int>(), sm.count2, b);
          f->prof.launches += 1;
        }
        if (f->F.is_mesh) {
          ProfScope ps(f->prof, Prof::FWD, ss);
          mesh::trace_paths_kernel<<<std::min(g, f->sm_count * 8), 256, 0, ss>>>(f->M, S, f->list.as<int>(), sm.count2,
                                                                                Pw);
          f->prof.launches += 1;
          f->prof.fwd_launches += 1;
        } else if ((rc = march(f, ms, Pw, f->list2.as<int>(), sm.stats + 0, ss,
                               fuse && b + 1 < cfg->bounces ? &tg : nullptr, S.want,
                               b < DDF_STAGE_BOUNCES ? sm.bmarch_rows() + b : nullptr, 0, lg_on ? &lg : nullptr,
                               b))) {
          return rc;
        }
        {
          ProfScope ps(f->prof, Prof::AFTER, ss);
          after_bounce_kernel<<<std::min(g, f->sm_count * 8), 256, 0, ss>>>(w, S, f->list.as<int>(), sm.count2);
          f->prof.launches += 1;
        }
      }
      {
        ProfScope ps(f->prof, Prof::FILM, ss);
        film_kernel<<<(n_own + 255) / 256, 256, 0, ss>>>(w, S, film);
        f->prof.launches += 1;
      }
      CUDA_TRY(cudaGetLastError());
      ++waves;
    }
    return DDF_OK;
  };
  // CUDA graph replay (cfg->graph): the captured loop is keyed by the field
  // generation, the buffer epoch, the camera and the config.  It writes the
  // field's own film buffer, so any caller accumulator can replay it.
  const bool use_graph = cfg->graph != 0 && !f->prof.on && !lg_on;
  std::vector<unsigned char> gkey;
  if (use_graph) {
    ddf_path_config_t kc = *cfg;
    kc.profile = 0;
    kc.graph = 0;
    const unsigned long long gen = f->gen;
    auto put = [&](const void* p, size_t n) { gkey.insert(gkey.end(), (const unsigned char*)p, (const unsigned char*)p + n); };
    put(&gen, sizeof gen);
    put(cam, sizeof(*cam));
    kc.tile_owner = nullptr;   // the table's contents, not its address, key the graph
    kc.stage_log = nullptr;
    put(&kc, sizeof kc);
    if (!owner.empty()) put(owner.data(), sizeof(int32_t) * owner.size());
  }
  auto epoch_key = [&]() {
    std::vector<unsigned char> k = gkey;
    k.insert(k.end(), (const unsigned char*)&g_buf_epoch, (const unsigned char*)&g_buf_epoch + sizeof g_buf_epoch);
    return k;
  };
  bool replayed = false;
  if (use_graph && f->graph_exec && f->graph_key == epoch_key()) {
    CUDA_TRY(cudaGraphLaunch(f->graph_exec, st));
    replayed = true;
    waves = f->graph_waves;
    f->prof.launches = f->graph_launches[0];
    f->prof.fwd_launches = f->graph_launches[1];
    f->prof.grad_launches = f->graph_launches[2];
    f->prof.fused_launches = f->graph_launches[3];
  } else {
    if (int rc = run_waves(st)) return rc;
    if (use_graph) {
      const uint64_t l0 = f->prof.launches, l1 = f->prof.fwd_launches, l2 = f->prof.grad_launches,
                     l3 = f->prof.fused_launches;
      const int w0 = waves;
      if (!f->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&f->cap_stream, cudaStreamNonBlocking));
      if (f->graph_exec) {
        cudaGraphExecDestroy(f->graph_exec);
        f->graph_exec = nullptr;
      }
      const std::vector<unsigned char> k = epoch_key();   // the eager run grew every buffer already
      cudaGraph_t graph = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(f->cap_stream, cudaStreamCaptureModeRelaxed));
      const int rc = run_waves(f->cap_stream);
      const cudaError_t ec = cudaStreamEndCapture(f->cap_stream, &graph);
      if (rc == DDF_OK && ec == cudaSuccess && graph && k == epoch_key()) {
        if (cudaGraphInstantiate(&f->graph_exec, graph, 0) == cudaSuccess) {
          f->graph_key = k;
          f->graph_waves = w0;
          f->graph_launches[0] = l0; f->graph_launches[1] = l1; f->graph_launches[2] = l2; f->graph_launches[3] = l3;
        } else {
          f->graph_exec = nullptr;
        }
      }
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();   // a failed capture only means no replay next time
      f->prof.launches = l0; f->prof.fwd_launches = l1; f->prof.grad_launches = l2; f->prof.fused_launches = l3;
      waves = w0;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(accum, film, sizeof(double) * n_pix, cudaMemcpyDeviceToDevice, st));
  if (f->prof.on) f->prof.marks[Prof::TOTAL].push_back({t_begin, f->prof.rec(st)});
  int host_small[32 + 2 * SMALL_U64];
  CUDA_TRY(cudaMemcpyAsync(host_small, f->small.p, sizeof(host_small), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const unsigned long long* hs64 = reinterpret_cast<const unsigned long long*>(host_small + 32);
  if (stats) {
    stats->forward_rows = hs64[0];
    stats->gradient_rows = hs64[1];
    stats->fused_rows = fuse ? hs64[3] : 0;
    stats->gradient_rows_executed = fuse ? hs64[4] : hs64[1];
    stats->fused_launches = f->prof.fused_launches;
    stats->ms_fused = f->prof.total_ms(Prof::FUSED);
    stats->degenerate = hs64[2];
    stats->path_samples = (uint64_t)n_own * cfg->spp;
    stats->waves = waves;
    stats->kernel_launches = f->prof.launches;
    stats->forward_launches = f->prof.fwd_launches;
    stats->gradient_launches = f->prof.grad_launches;
    stats->ms_forward = f->prof.total_ms(Prof::FWD);
    stats->ms_gradient = f->prof.total_ms(Prof::GRAD);
    stats->ms_compact = f->prof.total_ms(Prof::COMPACT);
    stats->graph_replayed = replayed ? 1 : 0;
    stats->ms_camera = f->prof.total_ms(Prof::CAMERA);
    stats->ms_roulette = f->prof.total_ms(Prof::ROULETTE);
    stats->ms_bounce = f->prof.total_ms(Prof::BOUNCE);
    stats->ms_after = f->prof.total_ms(Prof::AFTER);
    stats->ms_film = f->prof.total_ms(Prof::FILM);
    stats->ms_other = f->prof.total_ms(Prof::OTHER) + stats->ms_camera + stats->ms_roulette + stats->ms_bounce +
                      stats->ms_after + stats->ms_film;
    stats->ms_total = f->prof.total_ms(Prof::TOTAL);
    for (int j = 0; j < DDF_STAGE_STEPS; ++j) stats->primary_march_rows[j] = hs64[16 + j];
    for (int b = 0; b < DDF_STAGE_BOUNCES; ++b) {
      stats->bounce_alive_rows[b] = hs64[16 + DDF_STAGE_STEPS + b];
      stats->bounce_march_rows[b] = hs64[16 + DDF_STAGE_STEPS + DDF_STAGE_BOUNCES + b];
    }
  }
  if (host_small[18] & DEVERR_SIGN_RULE) return fail(DDF_ENUMERIC, "normal sign rule violated: n . dir >= 0");
  return DDF_OK;
}

int ddf_render_mode(ddf_field_t f, const ddf_camera_t* cam, const ddf_mode_config_t* cfg, double* out, void* stream) {
  if (!has_geometry(f)) return fail(DDF_EUSAGE, "field has no network");
  if (!cam || !cfg || !out) return fail(DDF_EUSAGE, "null argument");
  if (cfg->mode < 0 || cfg->mode > 2) return fail(DDF_EUSAGE, "unknown render mode");
  if (cam->width < 1 || cam->height < 1) return fail(DDF_EUSAGE, "film dimensions must be >= 1");
  const int64_t P64 = (int64_t)cam->width * cam->height;
  if (P64 > (1ll << 30)) return fail(DDF_EUSAGE, "film too large");
  const int P = (int)P64;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(f->device));
  if (int rc = ensure_small(f)) return rc;
  Small sm = small_of(f);
  f->prof.reset(false);
  CUDA_TRY(cudaMemsetAsync(f->small.p, 0, 4096, st));
  CUDA_TRY(f->st_o.ensure(sizeof(double) * 3 * P));
  CUDA_TRY(f->st_d.ensure(sizeof(double) * 3 * P));
  CUDA_TRY(f->st_tacc.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_texit.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_t.ensure(sizeof(double) * P));
  CUDA_TRY(f->st_hit.ensure(P));
  CUDA_TRY(f->st_march.ensure(P));
  CUDA_TRY(f->st_obj.ensure(sizeof(int) * P));
  CUDA_TRY(f->st_u34.ensure(sizeof(double) * 2 * P));
  CUDA_TRY(f->st_g3.ensure(sizeof(double) * 3 * P));
  CUDA_TRY(f->st_gdone.ensure(P));
  CUDA_TRY(f->st_want.ensure(P));
  CUDA_TRY(f->list.ensure(sizeof(int) * P));
  CUDA_TRY(f->list2.ensure(sizeof(int) * P));
  PathState S{};
  S.o = f->st_o.as<double>(); S.d = f->st_d.as<double>();
  S.t_acc = f->st_tacc.as<double>(); S.t_exit = f->st_texit.as<double>(); S.t = f->st_t.as<double>();
  S.hit = f->st_hit.as<uint8_t>(); S.march = f->st_march.as<uint8_t>();
  S.obj = f->st_obj.as<int>(); S.u34 = f->st_u34.as<double>(); S.g3 = f->st_g3.as<double>();
  MarchState ms{};
  ms.o = S.o; ms.d = S.d; ms.t_acc = S.t_acc; ms.t_exit = S.t_exit; ms.alive = S.march;
  ms.t_out = S.t; ms.hit = S.hit; ms.obj = S.obj; ms.u34 = S.u34;
  CamDev C{};
  for (int k = 0; k < 3; ++k) {
    C.pos[k] = cam->position[k]; C.fwd[k] = cam->forward[k]; C.right[k] = cam->right[k]; C.up[k] = cam->up_ortho[k];
  }
  C.tan_half = cam->tan_half; C.aspect = cam->aspect; C.W = cam->width; C.H = cam->height;
  const int g = (P + 255) / 256;
  camera_center_kernel<<<g, 256, 0, st>>>(f->F, C, S, P);
  CUDA_TRY(cudaGetLastError());
  // trace_batch (render.py:148,158,173)
  if (f->F.is_mesh) {
    mesh::trace_paths_kernel<<<g, 256, 0, st>>>(f->M, S, nullptr, nullptr, P);
    CUDA_TRY(cudaGetLastError());
  } else if (int rc = march(f, ms, P, f->list2.as<int>(), sm.stats + 0, st)) {
    return rc;
  }
  if (cfg->mode != 0) {
    // normals of the hit pixels (render.py:130-131)
    const int nobj = f->F.n_obj;
    if (int rc = compact_flags(f, S.hit, nobj > 1 ? S.obj : nullptr, P, std::max(1, nobj), f->list.as<int>(),
                               sm.seg, sm.count2, sm.stats + 1, st))
      return rc;
    if (f->F.is_mesh) {
      mesh::face_normal_kernel<<<std::min(g, f->sm_count * 8), 256, 0, st>>>(f->M, S, f->list.as<int>(), sm.count2);
      CUDA_TRY(cudaGetLastError());
    } else {
      GradOutOp op{};
      op.list = f->list.as<int>(); op.count = sm.count2; op.n = P;
      op.seg = nobj > 1 ? sm.seg : nullptr;
      op.S = S; op.backoff = f->F.backoff;
      if (int rc = run_mlp(f, f->F, op, P, true, st)) return rc;
    }
  }
  ModeDev m{};
  m.mode = cfg->mode; m.ambient = cfg->ambient;
  for (int k = 0; k < 3; ++k) { m.bg[k] = cfg->background[k]; m.light[k] = cfg->light_dir[k]; }
  m.albedo = cfg->albedo; m.env = cfg->env_radiance;
  mode_shade_kernel<<<g, 256, 0, st>>>(m, S, P, out, sm.err, sm.stats + 2);
  CUDA_TRY(cudaGetLastError());
  int host_small[32];
  CUDA_TRY(cudaMemcpyAsync(host_small, f->small.p, sizeof(host_small), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (host_small[18] & DEVERR_SIGN_RULE) return fail(DDF_ENUMERIC, "normal sign rule violated: n . dir >= 0");
  return DDF_OK;
}

namespace {
__global__ void rng_kernel(const PcgStream* st, const uint64_t* idx, int n, double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = pcg_single(*st, idx[j]);
}
}  // namespace

int ddf_rng_doubles(const uint64_t state[2], const uint64_t inc[2], const uint64_t* idx, int64_t n, double* out,
                    void* stream) {
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad count");
  if (n == 0) return DDF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  PcgStream hs;
  build_stream(state, inc, &hs);
  PcgStream* d = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&d, sizeof(hs), st));
  CUDA_TRY(cudaMemcpyAsync(d, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));
  rng_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(d, idx, (int)n, out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(d, st));
  CUDA_TRY(cudaStreamSynchronize(st));   // hs lives on this stack frame
  return DDF_OK;
}

int ddf_debug_trace(uint64_t* out, int32_t cap, int32_t reset) {
  if (!out || cap < 0) return -1;
  return engines::umma_debug_trace(reinterpret_cast<unsigned long long*>(out), cap, reset != 0);
}

int ddf_debug_counters(uint64_t* out16, int32_t reset) {
  unsigned long long h[16];
  engines::umma_debug_counters(h, reset != 0);
  for (int i = 0; i < 16; ++i) out16[i] = h[i];
  return DDF_OK;
}

int ddf_compact(const uint8_t* flags, int64_t n, int32_t* list, int32_t* count, void* stream) {
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad count");
  cudaStream_t st = (cudaStream_t)stream;
  // scratch is stream-ordered and per call, on the device that owns `flags`
  // (no process-wide buffers, nothing a captured render graph refers to)
  cudaPointerAttributes pa{};
  if (n > 0) {
    CUDA_TRY(cudaPointerGetAttributes(&pa, flags));
    if (pa.type == cudaMemoryTypeDevice) CUDA_TRY(cudaSetDevice(pa.device));
  }
  const int nb1 = std::max<int>(1, (int)((n + compact::OP_ITEMS - 1) / compact::OP_ITEMS));
  unsigned long long* state = nullptr;
  const size_t bytes = sizeof(unsigned long long) * (nb1 + compact::OP_STATE_EXTRA) + 2 * sizeof(int);
  CUDA_TRY(cudaMallocAsync((void**)&state, bytes, st));
  CUDA_TRY(cudaMemsetAsync(state, 0, sizeof(unsigned long long) * (nb1 + compact::OP_STATE_EXTRA), st));
  int* seg = reinterpret_cast<int*>(state + nb1 + compact::OP_STATE_EXTRA);
  compact::onepass_kernel<<<nb1, compact::NT, 0, st>>>(flags, nullptr, 0, (int)n, nb1, state, list, seg, count,
                                                        nullptr, nullptr, nullptr);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(state, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return DDF_OK;
}

int ddf_mesh_create(const double* vertices, int64_t n_vertices, const int32_t* faces, int64_t n_faces,
                    int32_t device, ddf_field_t* out) {
  if (!out || !vertices || !faces) return fail(DDF_EUSAGE, "null argument");
  if (n_vertices < 0 || n_faces < 0 || n_faces > (1ll << 28)) return fail(DDF_EDATA, "bad mesh sizes");
  if (n_faces == 0) return fail(DDF_EDATA, "cannot build a BVH over an empty mesh");   // mesh.py:98-99
  for (int64_t i = 0; i < 3 * n_faces; ++i)
    if (faces[i] < 0 || faces[i] >= n_vertices) return fail(DDF_EDATA, "face index out of range");   // mesh.py:33-34
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n_vertices; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], vertices[3 * i + k]);
      hi[k] = std::max(hi[k], vertices[3 * i + k]);
    }
  const double b6[6] = {lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]};
  ddf_field_t h = nullptr;
  if (int rc = ddf_field_create(1.0, b6, DDF_PREC_FP32, device, &h)) return rc;
  h->F.is_mesh = 1;
  if (int rc = build_mesh(h, vertices, n_vertices, faces, n_faces)) {
    ddf_field_destroy(h);
    return rc;
  }
  cudaError_t e = cudaMemcpy(h->F_dev, &h->F, sizeof(FieldDev), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    ddf_field_destroy(h);
    return fail(DDF_ECUDA, cudaGetErrorString(e));
  }
  *out = h;
  return DDF_OK;
}

int ddf_mesh_intersect(ddf_field_t f, const double* origins, const double* dirs, int64_t n, double t_min,
                       double t_max, int64_t* face, double* t, double* u, double* v, void* stream) {
  if (!f || !f->F.is_mesh) return fail(DDF_EUSAGE, "not a mesh field");
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad row count");
  if (n == 0) return DDF_OK;
  CUDA_TRY(cudaSetDevice(f->device));
  mesh::intersect_kernel<<<(int)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(f->M, origins, dirs, (int)n, t_min,
                                                                                 t_max, face, t, u, v);
  CUDA_TRY(cudaGetLastError());
  return DDF_OK;
}

int ddf_mesh_closest(ddf_field_t f, const double* points, int64_t n, double* out, void* stream) {
  if (!f || !f->F.is_mesh) return fail(DDF_EUSAGE, "not a mesh field");
  if (n < 0 || n > (1ll << 30)) return fail(DDF_EUSAGE, "bad point count");
  if (n == 0) return DDF_OK;
  CUDA_TRY(cudaSetDevice(f->device));
  mesh::closest_kernel<<<(int)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(f->M, points, (int)n, out);
  CUDA_TRY(cudaGetLastError());
  return DDF_OK;
}

int ddf_udf(ddf_field_t f, const double* points, int64_t n, int32_t n_dirs, int32_t polish, double* out,
            void* stream) {
  if (f && f->F.is_mesh) return ddf_mesh_closest(f, points, n, out, stream);   // exact backends (field.py:431-433)
  if (!f || f->F.n_obj == 0) return fail(DDF_EUSAGE, "field has no network");
  CUDA_TRY(cudaSetDevice(f->device));
  return udf_run(f, points, n, n_dirs, polish != 0, out, (cudaStream_t)stream);
}

int ddf_udf_grid(ddf_field_t f, const double bbox[6], int32_t resolution, int32_t n_dirs, int32_t polish,
                 double* out, void* stream) {
  if (!has_geometry(f)) return fail(DDF_EUSAGE, "field has no network");
  if (!bbox) return fail(DDF_EUSAGE, "null bbox");
  if (resolution < 8) return fail(DDF_EUSAGE, "resolution must be >= 8");   // recon.py:66-67
  if (resolution > 1024) return fail(DDF_EUSAGE, "resolution too large");
  CUDA_TRY(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = (int64_t)resolution * resolution * resolution;
  CUDA_TRY(f->udf_pts.ensure(sizeof(double) * 3 * n));
  udf::grid_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      f->udf_pts.as<double>(), resolution, bbox[0], bbox[1], bbox[2], bbox[3], bbox[4], bbox[5]);
  CUDA_TRY(cudaGetLastError());
  if (f->F.is_mesh) return ddf_mesh_closest(f, f->udf_pts.as<double>(), n, out, st);   // recon.py:61-81, exact
  return udf_run(f, f->udf_pts.as<double>(), n, n_dirs, polish != 0, out, st);
}

}  // extern "C"
