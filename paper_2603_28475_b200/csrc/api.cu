// api.cu — host side of libtac: the C ABI of include/tac.h.
//
// tac_create: validation, fp64 precompute of the rest shape (Dm^-1 rows, volumes,
// lumped masses), gel surface extraction, indenter BVHs (body frame,
// static, shared by all envs), fp64 marker location, device allocation in the
// env-fastest layout of internal.h.  tac_step: the launch sequence of SURVEY §3.3
// (rows a1-a9) on the caller's stream, no host synchronisation in fixed-iteration mode.
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <set>
#include <string>
#include <functional>
#include <vector>

#include "../../include/tac.h"
#include "internal.h"

using namespace tac;

struct tac_sim {
  Dev d;
  int device;
  std::vector<void*> allocs;
  std::string err;
  bool sticky = false;
  long long launches = 0;
  int max_iters, fixed_iters, check_every;
  // host copies for debug hooks
  std::vector<int> sv, st_flat, se_flat, ie_flat;
  std::vector<int> mk_tet, mk_idx;
  std::vector<double> mk_w;
  int* d_flag = nullptr;
  int* h_flag = nullptr;
  unsigned long long* d_dbg_cand = nullptr;
  int* d_dbg_cnt = nullptr;
  float* d_scratch = nullptr;  // [nv][3] host<->device staging
  tac::Profiler* prof = nullptr;
  // per-env material (tac_set_env_material): create-time base and the current values
  double E0 = 0, nu0 = 0, rho0 = 0, lbar = 0;
  bool kappa_fixed = false;
  unsigned long long step_count = 0;  // tac_step calls so far (pose-noise counter, R27)
  std::vector<double> thE, thNu, thRho, thMu;
  // CUDA graphs of the PNCG iteration loop: a chunk of n iterations (all K of the fixed mode,
  // check_every of the tolerance mode) is captured once per (h, anchor buffer) and replayed.
  // The Dev argument baked into the nodes differs between steps only in the anchor buffer
  // (double-buffered by the per-step sort), so two cached graphs cover every step.
  struct IterGraph {
    cudaGraphExec_t exec = nullptr;
    const void* anc = nullptr;
    double h = 0;
    int n = 0;
    bool fin = false;
    long long launches = 0;
    unsigned long long used = 0;  // LRU stamp
  } graphs[4];
  unsigned long long graph_clock = 0;
  // tolerance mode: one graph holding a WHILE node over (one PNCG iteration + k_loop_ctl), per
  // (anchor buffer, h, budget); the loop runs on the device until no env iterates or the
  // budget's last iteration is reached -- no host round trip inside a step
  struct WhileGraph {
    cudaGraphExec_t exec = nullptr;
    const void* anc = nullptr;
    double h = 0;
    int K = 0;
    long long launches_per_trip = 0;
  } wgraphs[2];
  bool use_while = true;     // TAC_NO_WHILE=1 at create: host-polled chunks instead (A/B)
  int* d_loop = nullptr;     // [1] iterations run by the WHILE loop of the current step
  long long while_per_trip = 0;  // launches per WHILE trip of the last step (0: no device loop)
  cudaStream_t cap = nullptr;  // capture stream (graphs are launched on the caller's stream)
  bool use_graphs = true;      // TAC_NO_GRAPH=1 at create disables (A/B measurements)
};

static thread_local std::string g_create_err;
static int g_tl_iter = -1;  // TAC_TIMELINE: the iteration of each step whose timeline is printed

namespace tac {
// per-kernel CUDA-event timing of the launches issued by tac_step / tac_markers
struct Profiler {
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[KID_COUNT];
  cudaEvent_t cur[KID_COUNT] = {};
  double ms[KID_COUNT] = {};
  long long cnt[KID_COUNT] = {};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void drain() {
    for (int k = 0; k < KID_COUNT; ++k) {
      for (auto& pr : pending[k]) {
        float t = 0.f;
        cudaEventSynchronize(pr.second);
        cudaEventElapsedTime(&t, pr.first, pr.second);
        ms[k] += t;
        cnt[k] += 1;
        pool.push_back(pr.first);
        pool.push_back(pr.second);
      }
      pending[k].clear();
    }
  }
  ~Profiler() {
    drain();
    for (auto e : pool) cudaEventDestroy(e);
  }
};
thread_local bool g_tl_on = false;
struct Timeline {
  cudaEvent_t start = nullptr;
  std::vector<std::pair<int, cudaEvent_t>> marks;
  std::vector<cudaStream_t> streams;
};
static Timeline g_tl;
void tl_mark(int kid, cudaStream_t s) {
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  g_tl.marks.push_back({kid, e});
  g_tl.streams.push_back(s);
}
static void tl_print() {  // end times (us from the iteration start) per launch and stream
  cudaEventSynchronize(g_tl.marks.empty() ? g_tl.start : g_tl.marks.back().second);
  cudaDeviceSynchronize();
  std::vector<cudaStream_t> ids;
  for (size_t i = 0; i < g_tl.marks.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, g_tl.start, g_tl.marks[i].second);
    int sid = (int)(std::find(ids.begin(), ids.end(), g_tl.streams[i]) - ids.begin());
    if (sid == (int)ids.size()) ids.push_back(g_tl.streams[i]);
    fprintf(stderr, "timeline stream %d %-22s end %8.1f us\n", sid, kernel_name(g_tl.marks[i].first), ms * 1e3);
    cudaEventDestroy(g_tl.marks[i].second);
  }
  cudaEventDestroy(g_tl.start);
  g_tl = Timeline{};
}
void prof_begin(int kid, cudaStream_t s) {
  cudaEvent_t e = g_prof->get();
  cudaEventRecord(e, s);
  g_prof->cur[kid] = e;
}
void prof_end(int kid, cudaStream_t s) {
  cudaEvent_t e = g_prof->get();
  cudaEventRecord(e, s);
  g_prof->pending[kid].push_back({g_prof->cur[kid], e});
}
}  // namespace tac

namespace {

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      sim->err = std::string(#x) + ": " + cudaGetErrorString(e_);               \
      sim->sticky = true;                                                       \
      return TAC_ECUDA;                                                         \
    }                                                                           \
  } while (0)

template <typename T>
tac_status upload(tac_sim* sim, const std::vector<T>& h, T** out) {
  size_t n = std::max<size_t>(1, h.size()) * sizeof(T);
  void* p = nullptr;
  if (cudaMalloc(&p, n) != cudaSuccess) { sim->err = "cudaMalloc failed"; return TAC_ENOMEM; }
  sim->allocs.push_back(p);
  if (!h.empty()) CK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = (T*)p;
  return TAC_OK;
}
template <typename T>
tac_status zalloc(tac_sim* sim, size_t n, T** out) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)) != cudaSuccess) {
    sim->err = "cudaMalloc failed (" + std::to_string(n * sizeof(T)) + " bytes)";
    return TAC_ENOMEM;
  }
  sim->allocs.push_back(p);
  CK(cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T)));
  *out = (T*)p;
  return TAC_OK;
}

typedef std::array<double, 3> V;
V sub(const V& a, const V& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
double det(const V& a, const V& b, const V& c) {  // det [a b c] (columns)
  return a[0] * (b[1] * c[2] - b[2] * c[1]) - b[0] * (a[1] * c[2] - a[2] * c[1]) + c[0] * (a[1] * b[2] - a[2] * b[1]);
}

// ---- BVH over indenter primitives (body frame), median split on the longest centroid axis ----
struct Build {
  std::vector<BNode>* nodes;
  std::vector<int>* prims;
  const std::vector<std::array<float, 6>>* box;  // prim boxes (lo, hi)
};
int build_node(Build& B, std::vector<int>& ids, int lo, int hi) {
  BNode n;
  for (int a = 0; a < 3; ++a) { n.lo[a] = INFINITY; n.hi[a] = -INFINITY; }
  float clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = lo; i < hi; ++i) {
    const auto& b = (*B.box)[ids[i]];
    for (int a = 0; a < 3; ++a) {
      n.lo[a] = std::min(n.lo[a], b[a]);
      n.hi[a] = std::max(n.hi[a], b[3 + a]);
      float c = 0.5f * (b[a] + b[3 + a]);
      clo[a] = std::min(clo[a], c);
      chi[a] = std::max(chi[a], c);
    }
  }
  int idx = (int)B.nodes->size();
  B.nodes->push_back(n);
  if (hi - lo <= kNodeLeaf) {
    (*B.nodes)[idx].left = -(int)B.prims->size() - 1;
    (*B.nodes)[idx].right = hi - lo;
    for (int i = lo; i < hi; ++i) B.prims->push_back(ids[i]);
    return idx;
  }
  int ax = 0;
  for (int a = 1; a < 3; ++a)
    if (chi[a] - clo[a] > chi[ax] - clo[ax]) ax = a;
  int mid = (lo + hi) / 2;
  std::nth_element(ids.begin() + lo, ids.begin() + mid, ids.begin() + hi, [&](int x, int y) {
    const auto& bx = (*B.box)[x];
    const auto& by = (*B.box)[y];
    float cx = bx[ax] + bx[3 + ax], cy = by[ax] + by[3 + ax];
    return cx < cy || (cx == cy && x < y);
  });
  int l = build_node(B, ids, lo, mid);
  int r = build_node(B, ids, mid, hi);
  (*B.nodes)[idx].left = l;
  (*B.nodes)[idx].right = r;
  return idx;
}
int build_bvh(std::vector<BNode>& nodes, std::vector<int>& prims, const std::vector<std::array<float, 6>>& box) {
  std::vector<int> ids(box.size());
  std::iota(ids.begin(), ids.end(), 0);
  Build B{&nodes, &prims, &box};
  if (ids.empty()) {  // empty tree: a node that never hits
    BNode n;
    for (int a = 0; a < 3; ++a) { n.lo[a] = INFINITY; n.hi[a] = -INFINITY; }
    n.left = -(int)prims.size() - 1;
    n.right = 0;
    nodes.push_back(n);
    return (int)nodes.size() - 1;
  }
  return build_node(B, ids, 0, (int)ids.size());
}

// per-env material tables from the current theta (padding lanes take env 0's values)
tac_status upload_env_material(tac_sim* sim, cudaStream_t stream) {
  const Dev& d = sim->d;
  std::vector<float> em(4 * (size_t)d.Es);
  std::vector<double> ed(2 * (size_t)d.Es);
  const double mu0 = sim->E0 / (2 * (1 + sim->nu0));
  for (int e = 0; e < d.Es; ++e) {
    const int s = e < d.E ? e : 0;
    const double E = sim->thE[s], nu = sim->thNu[s];
    const double mu = E / (2 * (1 + nu)), lam = E * nu / ((1 + nu) * (1 - 2 * nu));
    em[e] = (float)mu;
    em[d.Es + e] = (float)(lam + mu);
    em[2 * (size_t)d.Es + e] = (float)(sim->thRho[s] / sim->rho0);
    em[3 * (size_t)d.Es + e] = (float)(mu / mu0);
    ed[e] = sim->kappa_fixed ? d.kappa_phys : 0.2 * E * sim->lbar * sim->lbar / (12.25 * d.dhat);  // R4 per env
    ed[d.Es + e] = sim->thMu[s];
  }
  // ordered on `stream` behind the caller's queued work; the host staging vectors are freed on
  // return, so the copies must have landed first
  if (cudaMemcpyAsync(d.emat, em.data(), sizeof(float) * em.size(), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
      cudaMemcpyAsync(d.edbl, ed.data(), sizeof(double) * ed.size(), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess)
    return TAC_ECUDA;
  return TAC_OK;
}

float down(double x) { float f = (float)x; return (double)f > x ? std::nextafter(f, -INFINITY) : f; }
float up(double x) { float f = (float)x; return (double)f < x ? std::nextafter(f, INFINITY) : f; }

}  // namespace

extern "C" {

const char* tac_last_error(const tac_sim* sim) { return sim ? sim->err.c_str() : g_create_err.c_str(); }

tac_status tac_create(const tac_create_info* info, tac_sim** out) {
  if (!out) return TAC_EINVAL;
  *out = nullptr;
  g_create_err.clear();
  auto fail = [&](tac_status st, const std::string& m) { g_create_err = m; return st; };
  if (!info || !info->gel || !info->mat || !info->markers || !info->indenter || !info->params || !info->init_poses)
    return fail(TAC_EINVAL, "null pointer in tac_create_info");
  const tac_tet_mesh& G = *info->gel;
  const tac_tri_mesh& I = *info->indenter;
  const tac_marker_set& MS = *info->markers;
  const tac_solver_params& P = *info->params;
  const tac_material& MT = *info->mat;
  if (G.n_verts < 4 || G.n_tets < 1 || !G.rest_xyz || !G.tets || G.n_fixed < 0 || (G.n_fixed > 0 && !G.fixed))
    return fail(TAC_EINVAL, "invalid gel mesh");
  if (I.n_verts < 3 || I.n_tris < 1 || !I.rest_xyz || !I.tris) return fail(TAC_EINVAL, "invalid indenter mesh");
  if (info->n_envs < 1) return fail(TAC_EINVAL, "n_envs must be >= 1");
  if (!(MT.E > 0) || !(MT.nu >= 0 && MT.nu < 0.5) || !(MT.rho > 0) || !(MT.mu_f >= 0))
    return fail(TAC_EINVAL, "invalid material");
  if (!(P.dhat > 0) || !(P.bp_margin >= 0.5 * P.dhat) || !(P.ccd_s > 0 && P.ccd_s < 1) || !(P.k_t > 0) ||
      !(P.k_r > 0) || !(P.f_max > 0) || !(P.t_max > 0) || !(P.eps_v > 0) || P.max_iters < 1 || P.fixed_iters < 0 ||
      P.beta_rule < 0 || P.beta_rule > 3 || P.precond < 0 || P.precond > 1 || P.pose_al < 0 || P.pose_al > 1 ||
      P.ee_mollifier < 0 || P.ee_mollifier > 1 || P.dedup < 0 || P.dedup > 1)
    return fail(TAC_EINVAL, "invalid solver parameters");
  if (MS.rows * MS.cols < 1 || !MS.rest_xyz || (MS.mode != 0 && MS.mode != 1))
    return fail(TAC_EINVAL, "invalid marker set");
  int nv = G.n_verts, nt = G.n_tets, niv = I.n_verts, nit = I.n_tris, nm = MS.rows * MS.cols;
  std::vector<V> X(nv), Y(niv);
  for (int i = 0; i < nv; ++i) X[i] = {G.rest_xyz[3 * i], G.rest_xyz[3 * i + 1], G.rest_xyz[3 * i + 2]};
  for (int i = 0; i < niv; ++i) Y[i] = {I.rest_xyz[3 * i], I.rest_xyz[3 * i + 1], I.rest_xyz[3 * i + 2]};
  for (int i = 0; i < 4 * nt; ++i)
    if (G.tets[i] < 0 || G.tets[i] >= nv) return fail(TAC_EINVAL, "tet index out of range");
  for (int i = 0; i < 3 * nit; ++i)
    if (I.tris[i] < 0 || I.tris[i] >= niv) return fail(TAC_EINVAL, "indenter triangle index out of range");
  std::vector<unsigned char> vflag(nv, 0);
  for (int i = 0; i < G.n_fixed; ++i) {
    if (G.fixed[i] < 0 || G.fixed[i] >= nv) return fail(TAC_EINVAL, "fixed index out of range");
    vflag[G.fixed[i]] |= 1;
  }
  // rest shape: b_k = rows of Dm^-1 (k = 1..3), V_e = det(Dm)/6, lumped mass rho V_e / 4 per vertex
  std::vector<float4> tetb(3 * (size_t)nt);
  std::vector<int4> tets(nt);
  std::vector<double> massd(nv, 0.0), smud(nv, 0.0);
  for (int e = 0; e < nt; ++e) {
    const int* t = G.tets + 4 * e;
    tets[e] = make_int4(t[0], t[1], t[2], t[3]);
    V a = sub(X[t[1]], X[t[0]]), b = sub(X[t[2]], X[t[0]]), c = sub(X[t[3]], X[t[0]]);
    double D = det(a, b, c);
    if (!(D > 0)) return fail(TAC_EINVAL, "non-positive tet volume at tet " + std::to_string(e));
    // inverse of [a b c] (columns) by cofactors: row k of the inverse = (cross of the other two)/D
    V r0 = {(b[1] * c[2] - b[2] * c[1]) / D, (b[2] * c[0] - b[0] * c[2]) / D, (b[0] * c[1] - b[1] * c[0]) / D};
    V r1 = {(c[1] * a[2] - c[2] * a[1]) / D, (c[2] * a[0] - c[0] * a[2]) / D, (c[0] * a[1] - c[1] * a[0]) / D};
    V r2 = {(a[1] * b[2] - a[2] * b[1]) / D, (a[2] * b[0] - a[0] * b[2]) / D, (a[0] * b[1] - a[1] * b[0]) / D};
    double vol = D / 6.0;
    tetb[3 * e] = make_float4((float)r0[0], (float)r0[1], (float)r0[2], (float)vol);
    unsigned fixmask = 0;
    for (int k = 0; k < 4; ++k)
      if (vflag[t[k]] & 1) fixmask |= 1u << k;
    float fm;
    memcpy(&fm, &fixmask, sizeof(float));
    tetb[3 * e + 1] = make_float4((float)r1[0], (float)r1[1], (float)r1[2], fm);
    {  // state-independent part of the exact diagonal blocks: V_e mu |b_k|^2 per corner
      double mu_ = MT.E / (2 * (1 + MT.nu));
      V b[4] = {{-(r0[0] + r1[0] + r2[0]), -(r0[1] + r1[1] + r2[1]), -(r0[2] + r1[2] + r2[2])}, r0, r1, r2};
      for (int k = 0; k < 4; ++k) smud[t[k]] += vol * mu_ * (b[k][0] * b[k][0] + b[k][1] * b[k][1] + b[k][2] * b[k][2]);
    }
    tetb[3 * e + 2] = make_float4((float)r2[0], (float)r2[1], (float)r2[2], 0.f);
    for (int k = 0; k < 4; ++k) massd[t[k]] += MT.rho * vol / 4.0;
  }
  // gel surface: faces of exactly one tet, minus faces whose 3 vertices are all fixed
  std::map<std::array<int, 3>, int> fc;
  for (int e = 0; e < nt; ++e) {
    const int* t = G.tets + 4 * e;
    for (int skip = 0; skip < 4; ++skip) {
      std::array<int, 3> f;
      int n = 0;
      for (int k = 0; k < 4; ++k)
        if (k != skip) f[n++] = t[k];
      std::sort(f.begin(), f.end());
      fc[f] += 1;
    }
  }
  std::vector<std::array<int, 3>> st;
  std::set<int> svs;
  std::set<std::pair<int, int>> ses;
  for (auto& kv : fc) {
    if (kv.second != 1) continue;
    const auto& f = kv.first;
    if ((vflag[f[0]] & 1) && (vflag[f[1]] & 1) && (vflag[f[2]] & 1)) continue;
    st.push_back(f);
    for (int i = 0; i < 3; ++i) {
      svs.insert(f[i]);
      int a = f[i], b = f[(i + 1) % 3];
      ses.insert({std::min(a, b), std::max(a, b)});
    }
  }
  std::set<std::pair<int, int>> ies;
  for (int i = 0; i < nit; ++i)
    for (int k = 0; k < 3; ++k) {
      int a = I.tris[3 * i + k], b = I.tris[3 * i + (k + 1) % 3];
      ies.insert({std::min(a, b), std::max(a, b)});
    }
  tac_sim* sim = new tac_sim();  // value-initialised: every Dev field starts at 0
  sim->device = info->device;
  if (cudaSetDevice(info->device) != cudaSuccess) {
    delete sim;
    return fail(TAC_ECUDA, "cudaSetDevice failed");
  }
  sim->sv.assign(svs.begin(), svs.end());
  for (auto& f : st) for (int k = 0; k < 3; ++k) sim->st_flat.push_back(f[k]);
  for (auto& e : ses) { sim->se_flat.push_back(e.first); sim->se_flat.push_back(e.second); }
  for (auto& e : ies) { sim->ie_flat.push_back(e.first); sim->ie_flat.push_back(e.second); }
  for (int v : sim->sv) vflag[v] |= 2;
  // markers: barycentric in the lowest-index rest tet with all coordinates >= -1e-12 (R22)
  sim->mk_tet.assign(nm, -1);
  sim->mk_idx.assign(4 * nm, 0);
  sim->mk_w.assign(4 * nm, 0.0);
  for (int m = 0; m < nm; ++m) {
    V p = {MS.rest_xyz[3 * m], MS.rest_xyz[3 * m + 1], MS.rest_xyz[3 * m + 2]};
    if (MS.mode == 0) {
      for (int e = 0; e < nt; ++e) {
        const int* t = G.tets + 4 * e;
        V a = sub(X[t[1]], X[t[0]]), b = sub(X[t[2]], X[t[0]]), c = sub(X[t[3]], X[t[0]]), q = sub(p, X[t[0]]);
        double D = det(a, b, c);
        double l1 = det(q, b, c) / D, l2 = det(a, q, c) / D, l3 = det(a, b, q) / D;  // Cramer
        double l[4] = {1.0 - l1 - l2 - l3, l1, l2, l3};
        if (l[0] >= -1e-12 && l[1] >= -1e-12 && l[2] >= -1e-12 && l[3] >= -1e-12) {
          double s = 0;
          for (double& x : l) { x = std::max(0.0, x); s += x; }
          for (int k = 0; k < 4; ++k) { sim->mk_idx[4 * m + k] = t[k]; sim->mk_w[4 * m + k] = l[k] / s; }
          sim->mk_tet[m] = e;
          break;
        }
      }
      if (sim->mk_tet[m] < 0) {
        delete sim;
        return fail(TAC_EINVAL, "marker " + std::to_string(m) + " outside the gel mesh");
      }
    } else {
      int k = MS.k;
      if (k < 1 || k > 4 || (int)sim->sv.size() < k) { delete sim; return fail(TAC_EINVAL, "invalid kNN k"); }
      std::vector<std::pair<double, int>> dv;
      for (int v : sim->sv) {
        V q = sub(X[v], p);
        dv.push_back({std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]), v});
      }
      std::partial_sort(dv.begin(), dv.begin() + k, dv.end());
      for (int j = 0; j < 4; ++j) sim->mk_idx[4 * m + j] = dv[0].second;
      if (dv[0].first == 0.0) sim->mk_w[4 * m] = 1.0;
      else {
        double s = 0;
        for (int j = 0; j < k; ++j) s += 1.0 / dv[j].first;
        for (int j = 0; j < k; ++j) { sim->mk_idx[4 * m + j] = dv[j].second; sim->mk_w[4 * m + j] = (1.0 / dv[j].first) / s; }
      }
    }
  }
  // indenter BVHs (body frame): triangles, edges, vertices
  std::vector<std::array<float, 6>> btri(nit), bedge(ies.size()), bvert(niv);
  auto primbox = [&](const int* ids, int n) {
    std::array<float, 6> b;
    for (int a = 0; a < 3; ++a) {
      double lo = Y[ids[0]][a], hi = lo;
      for (int j = 1; j < n; ++j) { lo = std::min(lo, Y[ids[j]][a]); hi = std::max(hi, Y[ids[j]][a]); }
      b[a] = down(lo);
      b[3 + a] = up(hi);
    }
    return b;
  };
  for (int i = 0; i < nit; ++i) btri[i] = primbox(I.tris + 3 * i, 3);
  for (size_t i = 0; i < bedge.size(); ++i) bedge[i] = primbox(&sim->ie_flat[2 * i], 2);
  for (int i = 0; i < niv; ++i) { int id = i; bvert[i] = primbox(&id, 1); }
  std::vector<BNode> nodes;
  std::vector<int> prims;
  Dev& d = sim->d;
  d.root_tri = build_bvh(nodes, prims, btri);
  d.root_edge = build_bvh(nodes, prims, bedge);
  d.root_vert = build_bvh(nodes, prims, bvert);
  // Kuhn cells: groups of 6 tets sharing an edge (the cell diagonal 0-7) whose other corners
  // form the 6-cycle 1-3-2-6-4-5; relabelled to the canonical pattern (tet j = 0 -> 1<<p0 ->
  // (1<<p0)|(1<<p1) -> 7 for the j-th permutation p of the axes) with geometry deciding which
  // diagonal end is corner 0 and which axis each 1-bit corner lies along
  std::vector<int4> cell_v;
  std::vector<unsigned> cell_fix;
  std::vector<float4> cell_aa;  // axis-aligned cells: (1/s0, 1/s1, 1/s2, 1) with corner bit b along axis b
  std::vector<float4> cell_tb;
  std::vector<int> rest_tets;
  {
    static const int kTet[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};
    std::map<std::pair<int, int>, std::vector<int>> edge_tets;
    for (int e = 0; e < nt; ++e) {
      const int* t = G.tets + 4 * e;
      for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j) edge_tets[{std::min(t[i], t[j]), std::max(t[i], t[j])}].push_back(e);
    }
    std::vector<char> used(nt, 0);
    auto dist2 = [&](int p, int q) { V r = sub(X[p], X[q]); return r[0] * r[0] + r[1] * r[1] + r[2] * r[2]; };
    // candidate diagonals: edges shared by exactly 6 tets, longest first globally (a cell
    // diagonal, ~1.7 cells, is claimed before an interior axis edge, ~1 cell, whose link is
    // also a 6-cycle could take the same tets)
    std::vector<std::pair<double, std::pair<int, int>>> cands;
    for (auto& kv : edge_tets)
      if (kv.second.size() == 6) cands.push_back({-dist2(kv.first.first, kv.first.second), kv.first});
    std::sort(cands.begin(), cands.end());
    for (auto& cand : cands) {
      {
        {
          auto it = edge_tets.find(cand.second);
          const std::vector<int>& grp = it->second;
          bool free_ = true;
          for (int g : grp) free_ = free_ && !used[g];
          if (!free_) continue;
          int A = it->first.first, B = it->first.second;
          const bool dbg = getenv("TAC_DEBUG_CELLS") != nullptr;
          // non-diagonal corners of each tet
          std::vector<std::pair<int, int>> pairs;
          std::map<int, std::vector<int>> nb;
          for (int g : grp) {
            int o[2], n = 0;
            for (int k = 0; k < 4; ++k) {
              int v = G.tets[4 * g + k];
              if (v != A && v != B && n < 2) o[n++] = v;
            }
            if (n != 2) { n = -1; break; }
            pairs.push_back({o[0], o[1]});
            nb[o[0]].push_back(o[1]);
            nb[o[1]].push_back(o[0]);
          }
          if (pairs.size() != 6 || nb.size() != 6) { if (dbg) fprintf(stderr, "cell %d-%d: pairs %zu nb %zu\n", A, B, pairs.size(), nb.size()); continue; }
          bool cyc = true;
          for (auto& kv : nb) cyc = cyc && kv.second.size() == 2;
          if (!cyc) { if (dbg) fprintf(stderr, "cell %d-%d: cycle\n", A, B); continue; }
          // bipartition of the 6-cycle
          std::map<int, int> side;
          int start = nb.begin()->first, prev = -1, cur = start;
          for (int s = 0; s < 6; ++s) {
            side[cur] = s & 1;
            int nx = nb[cur][0] == prev ? nb[cur][1] : nb[cur][0];
            prev = cur;
            cur = nx;
          }
          if (cur != start || side.size() != 6) { if (dbg) fprintf(stderr, "cell %d-%d: closed\n", A, B); continue; }
          double m0[2] = {0, 0}, m1[2] = {0, 0};
          for (auto& kv : side) { m0[kv.second] += dist2(kv.first, A); m1[kv.second] += dist2(kv.first, B); }
          int one_bit = m0[0] < m0[1] ? 0 : 1;  // class nearer to corner 0
          int c0 = A, c7 = B;
          if (!(m1[1 - one_bit] < m1[one_bit])) {  // then A is corner 7
            c0 = B; c7 = A;
            one_bit = 1 - one_bit;
          }
          int lab[8] = {c0, -1, -1, -1, -1, -1, -1, c7};
          bool ok = true;
          std::map<int, int> bitof;  // 1-bit corner -> axis bit
          for (auto& kv : side) {
            if (kv.second != one_bit) continue;
            V d = sub(X[kv.first], X[c0]);
            int ax = (std::fabs(d[0]) >= std::fabs(d[1]) && std::fabs(d[0]) >= std::fabs(d[2])) ? 0
                     : (std::fabs(d[1]) >= std::fabs(d[2]) ? 1 : 2);
            if (lab[1 << ax] != -1) ok = false;
            lab[1 << ax] = kv.first;
            bitof[kv.first] = 1 << ax;
          }
          if (!ok) { if (dbg) fprintf(stderr, "cell %d-%d: axis\n", A, B); continue; }
          for (auto& kv : side) {
            if (kv.second == one_bit) continue;
            int l = bitof[nb[kv.first][0]] | bitof[nb[kv.first][1]];
            if (l == 0 || lab[l] != -1) ok = false;
            else lab[l] = kv.first;
          }
          for (int s = 0; s < 8; ++s) ok = ok && lab[s] >= 0;
          if (!ok) { if (dbg) fprintf(stderr, "cell %d-%d: twobit\n", A, B); continue; }
          // every canonical tet must be one of the group's tets
          std::set<std::array<int, 4>> have;
          for (int g : grp) {
            std::array<int, 4> q;
            for (int k = 0; k < 4; ++k) q[k] = G.tets[4 * g + k];
            std::sort(q.begin(), q.end());
            have.insert(q);
          }
          for (int jt = 0; jt < 6 && ok; ++jt) {
            std::array<int, 4> q;
            for (int k = 0; k < 4; ++k) q[k] = lab[kTet[jt][k]];
            std::sort(q.begin(), q.end());
            ok = have.count(q) > 0;
          }
          if (!ok) { if (dbg) fprintf(stderr, "cell %d-%d: canon\n", A, B); continue; }
          cell_v.push_back(make_int4(lab[0], lab[1], lab[2], lab[3]));
          cell_v.push_back(make_int4(lab[4], lab[5], lab[6], lab[7]));
          unsigned fm = 0;
          for (int s = 0; s < 8; ++s)
            if (vflag[lab[s]] & 1) fm |= 1u << s;
          cell_fix.push_back(fm);
          {  // axis-aligned box with corner bit b along coordinate axis b (signed edge s_b)?
            const V o = X[lab[0]];
            const V e[3] = {sub(X[lab[1]], o), sub(X[lab[2]], o), sub(X[lab[4]], o)};
            double len = 0;
            for (int b = 0; b < 3; ++b) len = std::max(len, std::fabs(e[b][b]));
            const double tol = 1e-9 * len;
            bool aa = len > 0;
            for (int b = 0; b < 3 && aa; ++b)
              for (int a = 0; a < 3; ++a)
                if (a != b && std::fabs(e[b][a]) > tol) aa = false;
            for (int sl = 0; sl < 8 && aa; ++sl)
              for (int a = 0; a < 3; ++a) {
                double want = o[a];
                for (int b = 0; b < 3; ++b)
                  if (sl & (1 << b)) want += e[b][a];
                if (std::fabs(X[lab[sl]][a] - want) > tol) aa = false;
              }
            // w = the common volume |s0 s1 s2| / 6 of the cell's six tets (> 0 marks the cell)
            cell_aa.push_back(aa ? make_float4((float)(1.0 / e[0][0]), (float)(1.0 / e[1][1]), (float)(1.0 / e[2][2]),
                                               (float)(std::fabs(e[0][0] * e[1][1] * e[2][2]) / 6.0))
                                 : make_float4(0.f, 0.f, 0.f, 0.f));
          }
          for (int jt = 0; jt < 6; ++jt) {  // b-vectors of the canonical corner order, |det|/6
            V a0 = X[lab[kTet[jt][0]]];
            V a = sub(X[lab[kTet[jt][1]]], a0), b = sub(X[lab[kTet[jt][2]]], a0), c = sub(X[lab[kTet[jt][3]]], a0);
            double D = det(a, b, c);
            V r0 = {(b[1] * c[2] - b[2] * c[1]) / D, (b[2] * c[0] - b[0] * c[2]) / D, (b[0] * c[1] - b[1] * c[0]) / D};
            V r1 = {(c[1] * a[2] - c[2] * a[1]) / D, (c[2] * a[0] - c[0] * a[2]) / D, (c[0] * a[1] - c[1] * a[0]) / D};
            V r2 = {(a[1] * b[2] - a[2] * b[1]) / D, (a[2] * b[0] - a[0] * b[2]) / D, (a[0] * b[1] - a[1] * b[0]) / D};
            cell_tb.push_back(make_float4((float)r0[0], (float)r0[1], (float)r0[2], (float)(std::fabs(D) / 6.0)));
            cell_tb.push_back(make_float4((float)r1[0], (float)r1[1], (float)r1[2], 0.f));
            cell_tb.push_back(make_float4((float)r2[0], (float)r2[1], (float)r2[2], 0.f));
          }
          for (int g : grp) used[g] = 1;
        }
      }
    }
    for (int e = 0; e < nt; ++e)
      if (!used[e]) rest_tets.push_back(e);
  }
  // cell rows: chains of cells along corner bit 0 (cell k+1's corners 0, 2, 4, 6 are cell k's
  // 1, 3, 5, 7), cells reordered chain by chain and cut into segments of <= seg_len cells; the
  // row-marching gradient pass carries the shared face's u and accumulators from one cell to
  // the next (half the corner loads and red.adds of one cell at a time)
  std::vector<int2> cell_seg;
  {
    const int ncell = (int)cell_fix.size();
    auto corner = [&](int c, int k) {
      const int4 q = cell_v[2 * c + (k >> 2)];
      const int r = k & 3;
      return r == 0 ? q.x : r == 1 ? q.y : r == 2 ? q.z : q.w;
    };
    std::map<int, int> by0;
    for (int c = 0; c < ncell; ++c) by0[corner(c, 0)] = c;
    std::vector<int> nxt(ncell, -1), has_prev(ncell, 0);
    for (int c = 0; c < ncell; ++c) {
      auto it = by0.find(corner(c, 1));
      if (it == by0.end()) continue;
      const int c2 = it->second;
      bool ok = c2 != c;
      for (int k = 0; k < 8 && ok; k += 2) ok = corner(c2, k) == corner(c, k + 1);
      if (ok && !has_prev[c2]) { nxt[c] = c2; has_prev[c2] = 1; }
    }
    std::vector<int> order;
    std::vector<char> seen(ncell, 0);
    const int seg_len = std::min(kRowSegMax, getenv("TAC_ROW_SEG") ? std::max(1, atoi(getenv("TAC_ROW_SEG"))) : 10);
    auto chain = [&](int h) {
      int len = 0;
      for (int c = h; c >= 0 && !seen[c]; c = nxt[c]) { seen[c] = 1; order.push_back(c); ++len; }
      // split into near-equal segments of <= seg_len cells
      const int base = (int)order.size() - len, nsg = (len + seg_len - 1) / seg_len;
      for (int k = 0, at = 0; k < nsg; ++k) {
        const int n = (len - at) / (nsg - k);
        cell_seg.push_back(make_int2(base + at, n));
        at += n;
      }
    };
    for (int c = 0; c < ncell; ++c)
      if (!has_prev[c]) chain(c);
    for (int c = 0; c < ncell; ++c)
      if (!seen[c]) chain(c);  // (cycles cannot occur on a pad; kept total)
    std::vector<int4> v2(cell_v.size());
    std::vector<unsigned> f2(cell_fix.size());
    std::vector<float4> a2(cell_aa.size()), t2(cell_tb.size());
    for (int k = 0; k < ncell; ++k) {
      const int c = order[k];
      v2[2 * k] = cell_v[2 * c]; v2[2 * k + 1] = cell_v[2 * c + 1];
      f2[k] = cell_fix[c];
      a2[k] = cell_aa[c];
      for (int j = 0; j < 18; ++j) t2[18 * k + j] = cell_tb[18 * c + j];
    }
    cell_v.swap(v2); cell_fix.swap(f2); cell_aa.swap(a2); cell_tb.swap(t2);
  }
  // element tiles: Morton order of tet centroids, greedy cut at kTileT tets / kTileV
  // vertices, then greedy rounds of <= kTileW vertex-disjoint tets
  std::vector<int> tile_vstart{0}, tile_verts, tile_tstart{0}, tile_rstart{0};
  std::vector<unsigned char> tile_vfl;
  std::vector<uchar4> tile_tv;
  std::vector<float4> tile_tb;
  std::vector<short> tile_sched;
  {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (auto& x : X) for (int c = 0; c < 3; ++c) { lo[c] = std::min(lo[c], x[c]); hi[c] = std::max(hi[c], x[c]); }
    auto spread = [](unsigned v) {  // 10 bits -> every third bit
      v &= 1023u;
      v = (v | (v << 16)) & 0x030000FFu;
      v = (v | (v << 8)) & 0x0300F00Fu;
      v = (v | (v << 4)) & 0x030C30C3u;
      v = (v | (v << 2)) & 0x09249249u;
      return v;
    };
    std::vector<std::pair<unsigned, int>> order(nt);
    for (int e = 0; e < nt; ++e) {
      unsigned q[3];
      for (int c = 0; c < 3; ++c) {
        double m = 0;
        for (int k = 0; k < 4; ++k) m += X[G.tets[4 * e + k]][c];
        m /= 4;
        q[c] = (unsigned)std::min(1023.0, std::max(0.0, (m - lo[c]) / std::max(1e-30, hi[c] - lo[c]) * 1023.0));
      }
      order[e] = {spread(q[0]) | (spread(q[1]) << 1) | (spread(q[2]) << 2), e};
    }
    std::sort(order.begin(), order.end());
    std::vector<int> vtile(nv, -1), vcount_tiles(nv, 0), vlocal(nv, -1);
    std::vector<std::vector<int>> tiles;
    {
      std::vector<int> cur;
      std::set<int> cv;
      for (auto& pr : order) {
        int e = pr.second;
        std::set<int> add;
        for (int k = 0; k < 4; ++k)
          if (!cv.count(G.tets[4 * e + k])) add.insert(G.tets[4 * e + k]);
        if (!cur.empty() && ((int)cur.size() >= kTileT || (int)(cv.size() + add.size()) > kTileV)) {
          tiles.push_back(cur);
          cur.clear();
          cv.clear();
          for (int k = 0; k < 4; ++k) add.insert(G.tets[4 * e + k]);
        }
        cur.push_back(e);
        cv.insert(add.begin(), add.end());
      }
      if (!cur.empty()) tiles.push_back(cur);
    }
    // how many tiles touch each vertex (exclusive vertices can be flushed without atomics)
    for (size_t ti = 0; ti < tiles.size(); ++ti) {
      std::set<int> vs;
      for (int e : tiles[ti]) for (int k = 0; k < 4; ++k) vs.insert(G.tets[4 * e + k]);
      for (int v : vs) vcount_tiles[v] += 1;
    }
    for (size_t ti = 0; ti < tiles.size(); ++ti) {
      std::vector<int> verts;
      for (int e : tiles[ti]) for (int k = 0; k < 4; ++k) {
        int v = G.tets[4 * e + k];
        if (vlocal[v] < 0) { vlocal[v] = (int)verts.size(); verts.push_back(v); }
      }
      for (int v : verts) {
        tile_verts.push_back(v);
        tile_vfl.push_back((unsigned char)((vflag[v] & 1) | (vcount_tiles[v] == 1 ? 2 : 0)));
      }
      tile_vstart.push_back((int)tile_verts.size());
      for (int e : tiles[ti]) {
        const int* t = G.tets + 4 * e;
        tile_tv.push_back(make_uchar4((unsigned char)vlocal[t[0]], (unsigned char)vlocal[t[1]],
                                      (unsigned char)vlocal[t[2]], (unsigned char)vlocal[t[3]]));
        for (int r = 0; r < 3; ++r) tile_tb.push_back(tetb[3 * e + r]);
      }
      tile_tstart.push_back((int)tile_tv.size());
      // rounds: greedy, each round <= kTileW tets with pairwise disjoint vertices
      std::vector<int> left(tiles[ti].size());
      std::iota(left.begin(), left.end(), 0);
      while (!left.empty()) {
        std::vector<int> round, rest;
        std::set<int> used;
        for (int li : left) {
          const int* t = G.tets + 4 * tiles[ti][li];
          bool ok = (int)round.size() < kTileW;
          for (int k = 0; k < 4 && ok; ++k) ok = !used.count(t[k]);
          if (ok) {
            round.push_back(li);
            for (int k = 0; k < 4; ++k) used.insert(t[k]);
          } else {
            rest.push_back(li);
          }
        }
        for (int wslot = 0; wslot < kTileW; ++wslot)
          tile_sched.push_back(wslot < (int)round.size() ? (short)round[wslot] : (short)-1);
        left.swap(rest);
      }
      tile_rstart.push_back((int)tile_sched.size() / kTileW);
      for (int v : verts) vlocal[v] = -1;
    }
  }
  // sizes and parameters
  d.nv = nv; d.nt = nt; d.nsv = (int)sim->sv.size(); d.nse = (int)ses.size(); d.nst = (int)st.size();
  d.niv = niv; d.nie = (int)ies.size(); d.nit = nit; d.nm = nm;
  d.E = info->n_envs;
  d.Es = (d.E + 31) / 32 * 32;
  d.kmax = P.max_candidates > 0 ? P.max_candidates : 32768;
  d.amax = P.max_anchors > 0 ? P.max_anchors : 4096;
  if (d.amax > 16384) {  // the per-step anchor sort holds next_pow2(max_anchors) keys in shared memory
    delete sim;
    return fail(TAC_EINVAL, "max_anchors > 16384");
  }
  d.mu = (float)(MT.E / (2 * (1 + MT.nu)));
  double lam = MT.E * MT.nu / ((1 + MT.nu) * (1 - 2 * MT.nu));
  d.lam2 = (float)(lam + MT.E / (2 * (1 + MT.nu)));
  d.mu_f = MT.mu_f;
  d.rho_max = 0;
  for (auto& y : Y) d.rho_max = std::max(d.rho_max, std::sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2]));
  d.dhat = P.dhat; d.eps_v = P.eps_v; d.tol_x = P.tol_x; d.k_t = P.k_t; d.k_r = P.k_r; d.f_max = P.f_max;
  d.t_max = P.t_max; d.ccd_s = P.ccd_s; d.bp_margin = P.bp_margin; d.c1 = P.c1; d.eps_E = P.eps_E;
  d.kappa_phys = P.kappa_phys;
  if (!(d.kappa_phys > 0)) {  // R4 default: 0.2 E lbar^2 / (12.25 dhat), lbar = mean gel surface edge length
    double sl = 0;
    for (auto& e : ses) { V q = sub(X[e.first], X[e.second]); sl += std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]); }
    double lbar = ses.empty() ? 1e-3 : sl / ses.size();
    d.kappa_phys = 0.2 * MT.E * lbar * lbar / (12.25 * P.dhat);
    sim->lbar = lbar;
  } else {
    sim->kappa_fixed = true;
  }
  sim->E0 = MT.E; sim->nu0 = MT.nu; sim->rho0 = MT.rho;
  sim->thE.assign(d.E, MT.E); sim->thNu.assign(d.E, MT.nu); sim->thRho.assign(d.E, MT.rho); sim->thMu.assign(d.E, MT.mu_f);
  if (d.nsv >= 16384 || niv >= 16384) {  // candidate corner ids are packed 14 bit + the kind (Dev::ccorn)
    delete sim;
    return fail(TAC_EINVAL, "more than 16383 gel-surface or indenter vertices");
  }
  d.compact = getenv("TAC_NO_COMPACT") ? 0 : (getenv("TAC_COMPACT_LANES") ? atoi(getenv("TAC_COMPACT_LANES")) : 16);
  d.remap_blocks = getenv("TAC_REMAP_BLOCKS") ? std::max(0, atoi(getenv("TAC_REMAP_BLOCKS"))) : 512;
  d.contact_bps = getenv("TAC_CONTACT_BPS") ? std::max(1, atoi(getenv("TAC_CONTACT_BPS"))) : 8;
  d.contact_smem = contact_smem_bytes(d.nsv, niv);
  if (d.contact_smem == 0) {
    delete sim;
    return fail(TAC_EINVAL, "gel surface + indenter too large for the shared-memory staged contact passes");
  }
  kernels_init(d.contact_smem);
  d.pose_al = P.pose_al;
  d.ee_moll = P.ee_mollifier;
  d.dedup = P.dedup;
  d.beta_rule = P.beta_rule; d.precond = P.precond; d.max_halv = P.max_halvings; d.stagnation = P.stagnation;
  d.fixed_iters = P.fixed_iters;
  for (int a = 0; a < 3; ++a) { d.t1[a] = MS.t1[a]; d.t2[a] = MS.t2[a]; d.nrm[a] = MS.n[a]; }
  if (6.0 * nv * (double)d.Es >= 4294967296.0) { delete sim; return fail(TAC_EINVAL, "n_verts x n_envs too large for 32-bit offsets"); }
  sim->max_iters = P.max_iters;
  sim->fixed_iters = P.fixed_iters;
  sim->check_every = P.check_every > 0 ? P.check_every : 25;
  if (getenv("TAC_NO_GRAPH")) sim->use_graphs = false;
  if (getenv("TAC_NO_WHILE")) sim->use_while = false;
  if (getenv("TAC_TIMELINE") && P.fixed_iters > 0) {  // measurement only: direct launches
    sim->use_graphs = false;
    g_tl_iter = P.fixed_iters / 2;
  }
  if (getenv("TAC_TIMELINE_ITER")) {  // measurement only: that iteration of every launched chunk
    sim->use_graphs = false;
    g_tl_iter = atoi(getenv("TAC_TIMELINE_ITER"));
  }
  // device upload
  std::vector<float4> Xf(nv), Yf(niv);
  for (int i = 0; i < nv; ++i) Xf[i] = make_float4((float)X[i][0], (float)X[i][1], (float)X[i][2], 0.f);
  for (int i = 0; i < niv; ++i)
    Yf[i] = make_float4((float)Y[i][0], (float)Y[i][1], (float)Y[i][2],
                        (float)std::sqrt(Y[i][0] * Y[i][0] + Y[i][1] * Y[i][1] + Y[i][2] * Y[i][2]));
  std::vector<float> massf(nv), smuf(nv);
  for (int i = 0; i < nv; ++i) { massf[i] = (float)massd[i]; smuf[i] = (float)smud[i]; }
  std::vector<int2> se2, ie2;
  for (auto& e : ses) se2.push_back(make_int2(e.first, e.second));
  for (auto& e : ies) ie2.push_back(make_int2(e.first, e.second));
  std::vector<int4> st4, it4, st4l;
  std::vector<int2> se2l;
  std::vector<int> sidx_h(nv, -1);
  {
    std::vector<int> sloc(nv, -1);
    for (size_t i = 0; i < sim->sv.size(); ++i) sloc[sim->sv[i]] = (int)i;
    sidx_h = sloc;
    for (auto& f : st) st4l.push_back(make_int4(sloc[f[0]], sloc[f[1]], sloc[f[2]], 0));
    for (auto& e2 : ses) se2l.push_back(make_int2(sloc[e2.first], sloc[e2.second]));
  }
  for (auto& f : st) st4.push_back(make_int4(f[0], f[1], f[2], 0));
  for (int i = 0; i < nit; ++i) it4.push_back(make_int4(I.tris[3 * i], I.tris[3 * i + 1], I.tris[3 * i + 2], 0));
  std::vector<int4> mki(nm);
  std::vector<float4> mkw(nm);
  for (int m = 0; m < nm; ++m) {
    mki[m] = make_int4(sim->mk_idx[4 * m], sim->mk_idx[4 * m + 1], sim->mk_idx[4 * m + 2], sim->mk_idx[4 * m + 3]);
    mkw[m] = make_float4((float)sim->mk_w[4 * m], (float)sim->mk_w[4 * m + 1], (float)sim->mk_w[4 * m + 2],
                         (float)sim->mk_w[4 * m + 3]);
  }
  tac_status rc = TAC_OK;
#define UP(vec, dst)                                  \
  do {                                                \
    auto* tmp_ = (std::remove_const<std::remove_pointer<decltype(dst)>::type>::type*)nullptr; \
    rc = upload(sim, vec, &tmp_);                      \
    if (rc) goto fail;                                \
    dst = tmp_;                                       \
  } while (0)
  {
    UP(tets, d.tets);
    UP(tetb, d.tetb);
    UP(Xf, d.X);
    {
      std::vector<float4> Xs(sim->sv.size());  // surface-ordered rest positions (staged passes)
      for (size_t i = 0; i < sim->sv.size(); ++i) Xs[i] = Xf[sim->sv[i]];
      UP(Xs, d.Xs);
    }
    UP(massf, d.mass);
    UP(smuf, d.smu);
    UP(vflag, d.vflag);
    UP(sim->sv, d.sv);
    {
      std::vector<int> svfree(sim->sv.size());  // surface-local id -> free gel vertex id, -1 if fixed
      for (size_t i = 0; i < sim->sv.size(); ++i) svfree[i] = (vflag[sim->sv[i]] & 1) ? -1 : sim->sv[i];
      UP(svfree, d.svfree);
    }
    UP(se2, d.se);
    UP(st4, d.st);
    UP(se2l, d.se_l);
    UP(st4l, d.st_l);
    UP(sidx_h, d.sidx);
    UP(Yf, d.Y);
    UP(ie2, d.ie);
    UP(it4, d.it);
    {
      // 4-wide (child-box) form of the three BVHs: two binary levels collapsed into one 128-byte
      // node holding up to four children's boxes and refs (>= 0 internal, < 0 leaf: -1 - (first
      // prim << 3 | count)); empty slots never hit.  Wide nodes 0, 1, 2 are virtual roots (tri,
      // edge, vert) whose child 0 is the tree root.  Half the depth of the binary tree: a query
      // pays half the dependent node loads.
      std::vector<float4> wide(kBvhF4 * 3);
      auto put_wide = [&](int w, const float (*lo)[3], const float (*hi)[3], const int* ref) {
        for (int j = 0; j < kBvhW; j += 2) {  // children j, j+1: 12 floats in 3 float4
          wide[kBvhF4 * w + 3 * (j / 2)] = make_float4(lo[j][0], lo[j][1], lo[j][2], hi[j][0]);
          wide[kBvhF4 * w + 3 * (j / 2) + 1] = make_float4(hi[j][1], hi[j][2], lo[j + 1][0], lo[j + 1][1]);
          wide[kBvhF4 * w + 3 * (j / 2) + 2] = make_float4(lo[j + 1][2], hi[j + 1][0], hi[j + 1][1], hi[j + 1][2]);
        }
        for (int j = 0; j < kBvhW; j += 4) {  // refs, four per float4
          float rf[4];
          memcpy(rf, ref + j, sizeof(rf));
          wide[kBvhF4 * w + 3 * kBvhW / 2 + j / 4] = make_float4(rf[0], rf[1], rf[2], rf[3]);
        }
      };
      auto leaf_ref = [&](int k) { return -1 - (((-nodes[k].left - 1) << 3) | nodes[k].right); };
      std::function<int(int)> make_wide = [&](int k) -> int {  // binary internal node k -> wide index
        // children: expand internal descendants breadth-first while they fit in kBvhW slots
        std::vector<int> ch = {nodes[k].left, nodes[k].right};
        for (size_t j = 0; j < ch.size() && (int)ch.size() < kBvhW;) {
          if (nodes[ch[j]].left >= 0) {
            const int c = ch[j];
            ch.erase(ch.begin() + j);
            ch.push_back(nodes[c].left);
            ch.push_back(nodes[c].right);
          } else {
            ++j;
          }
        }
        const int w = (int)wide.size() / kBvhF4;
        wide.resize(wide.size() + kBvhF4);
        float lo[kBvhW][3], hi[kBvhW][3];
        int ref[kBvhW];
        for (int j = 0; j < kBvhW; ++j) {
          for (int t = 0; t < 3; ++t) { lo[j][t] = INFINITY; hi[j][t] = -INFINITY; }
          ref[j] = -1;  // empty leaf (never reached: its box never overlaps)
        }
        for (size_t j = 0; j < ch.size(); ++j) {
          const BNode& n = nodes[ch[j]];
          for (int t = 0; t < 3; ++t) { lo[j][t] = n.lo[t]; hi[j][t] = n.hi[t]; }
          ref[j] = n.left >= 0 ? make_wide(ch[j]) : leaf_ref(ch[j]);
        }
        put_wide(w, lo, hi, ref);
        return w;
      };
      const int roots[3] = {d.root_tri, d.root_edge, d.root_vert};
      for (int t = 0; t < 3; ++t) {  // virtual root t: child 0 = the tree's root, the rest empty
        const BNode& n = nodes[roots[t]];
        float lo[kBvhW][3], hi[kBvhW][3];
        int ref[kBvhW];
        for (int j = 0; j < kBvhW; ++j) {
          for (int q = 0; q < 3; ++q) { lo[j][q] = INFINITY; hi[j][q] = -INFINITY; }
          ref[j] = -1;
        }
        for (int q = 0; q < 3; ++q) { lo[0][q] = n.lo[q]; hi[0][q] = n.hi[q]; }
        ref[0] = n.left >= 0 ? make_wide(roots[t]) : leaf_ref(roots[t]);
        put_wide(t, lo, hi, ref);
      }
      UP(wide, d.bvhw);
    }
    UP(prims, d.bvh_prims);
    {
      // per-prim body-frame boxes in leaf order (lo.xyz | prim id bits, hi.xyz): the exact
      // min / max of the float Y the kernels use, so the leaf test needs one load per prim
      std::vector<float4> pbox(2 * prims.size());
      const int nie_ = (int)ies.size();
      for (size_t p = 0; p < prims.size(); ++p) {
        const int prim = prims[p];
        int ids[3], n;
        if ((int)p < nit) { ids[0] = I.tris[3 * prim]; ids[1] = I.tris[3 * prim + 1]; ids[2] = I.tris[3 * prim + 2]; n = 3; }
        else if ((int)p < nit + nie_) { ids[0] = sim->ie_flat[2 * prim]; ids[1] = sim->ie_flat[2 * prim + 1]; n = 2; }
        else { ids[0] = prim; n = 1; }
        float lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
          auto comp = [&](int v) { return a == 0 ? Yf[v].x : (a == 1 ? Yf[v].y : Yf[v].z); };
          lo[a] = hi[a] = comp(ids[0]);
          for (int j = 1; j < n; ++j) { lo[a] = std::min(lo[a], comp(ids[j])); hi[a] = std::max(hi[a], comp(ids[j])); }
        }
        int bits = prim;
        float fb;
        memcpy(&fb, &bits, sizeof(float));
        pbox[2 * p] = make_float4(lo[0], lo[1], lo[2], fb);
        pbox[2 * p + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
      }
      UP(pbox, d.bvh_pbox);
    }
    UP(mki, d.mk_idx);
    UP(mkw, d.mk_w);
    UP(tile_vstart, d.tile_vstart);
    UP(tile_verts, d.tile_verts);
    UP(tile_vfl, d.tile_vfl);
    UP(tile_tstart, d.tile_tstart);
    UP(tile_tv, d.tile_tv);
    UP(tile_tb, d.tile_tb);
    UP(tile_rstart, d.tile_rstart);
    UP(tile_sched, d.tile_sched);
    UP(cell_v, d.cell_v);
    UP(cell_fix, d.cell_fix);
    UP(cell_aa, d.cell_aa);
    d.cells_all_aa = !cell_aa.empty();
    for (auto& a : cell_aa) d.cells_all_aa = d.cells_all_aa && a.w > 0.f;
    if (getenv("TAC_DEBUG_CELLS")) {
      size_t naa = 0;
      for (auto& a : cell_aa) naa += a.w != 0.f;
      fprintf(stderr, "cells: %zu, axis-aligned (bit b along axis b): %zu\n", cell_aa.size(), naa);
    }
    UP(cell_tb, d.cell_tb);
    UP(cell_seg, d.cell_seg);
    d.nseg = (int)cell_seg.size();
    d.rows = d.cells_all_aa && !getenv("TAC_NO_ROWS");
    UP(rest_tets, d.rest_tets);
    d.ncells = (int)cell_fix.size();
    d.nrest = (int)rest_tets.size();
    d.ntiles = (int)tile_vstart.size() - 1;
    size_t nvec = 3 * (size_t)nv * d.Es;
    if ((rc = zalloc(sim, nvec, &d.u)) || (rc = zalloc(sim, nvec, &d.ut)) || (rc = zalloc(sim, nvec, &d.vt)) ||
        (rc = zalloc(sim, nvec, &d.uh)) || (rc = zalloc(sim, nvec, &d.g)) || (rc = zalloc(sim, nvec, &d.gp)) ||
        (rc = zalloc(sim, nvec, &d.p)) || (rc = zalloc(sim, nvec, &d.Pg)) || (rc = zalloc(sim, 2 * nvec, &d.D)) || (rc = zalloc(sim, (size_t)d.E, &d.es)) ||
        (rc = zalloc(sim, 4 * (size_t)d.Es, &d.emat)) || (rc = zalloc(sim, 2 * (size_t)d.Es, &d.edbl)) ||
        (rc = zalloc(sim, (size_t)kNAcc * d.Es, &d.acc)) || (rc = zalloc(sim, (size_t)kNAccU * d.Es, &d.accu)) ||
        (rc = zalloc(sim, (size_t)d.Es, &d.dalpha)) || (rc = zalloc(sim, (size_t)d.Es, &d.beta)) ||
        (rc = zalloc(sim, (size_t)d.Es, &d.run)) || (rc = zalloc(sim, (size_t)d.Es, &d.alist)) ||
        (rc = zalloc(sim, (size_t)d.Es / 32 + 1, &d.glist)) || (rc = zalloc(sim, (size_t)2, &d.anum)) ||
        (rc = zalloc(sim, (size_t)1, &d.adone)) || (rc = zalloc(sim, (size_t)d.Es, &d.pcf)) ||
        (rc = zalloc(sim, 2 * (size_t)d.E * d.kmax, &d.cand)) || (rc = zalloc(sim, (size_t)d.E, &d.lbuf)) || (rc = zalloc(sim, 2 * (size_t)d.E * d.kmax, &d.cgeo)) || (rc = zalloc(sim, (size_t)d.E * d.kmax, &d.cgap)) || (rc = zalloc(sim, 2 * (size_t)d.E * d.kmax, &d.ccorn)) || (rc = zalloc(sim, (size_t)d.E * d.kmax, &d.ncorn)) || (rc = zalloc(sim, 2 * (size_t)d.E, &d.ncand)) || (rc = zalloc(sim, 3 * (size_t)d.E * d.kmax, &d.nearl)) ||
        (rc = zalloc(sim, 3 * (size_t)d.E, &d.nnear)) ||
        (rc = zalloc(sim, 6 * (size_t)std::max(1, d.nsv) * d.Es, &d.Dcon)) ||
        (rc = zalloc(sim, d.dedup ? (size_t)kDedupSlots * d.Es : 1, &d.dtab)) ||
        (rc = zalloc(sim, (size_t)std::max(1, d.nsv) * d.Es, &d.usurf)) || (rc = zalloc(sim, (size_t)std::max(1, d.nsv) * d.Es, &d.psurf)) ||
        (rc = zalloc(sim, (size_t)d.E * d.amax, &d.anc)) || (rc = zalloc(sim, (size_t)d.E * d.amax, &d.anc2)) || (rc = zalloc(sim, (size_t)d.E * d.amax, &d.anc_f1)) || (rc = zalloc(sim, (size_t)d.E, &d.nanc)) || (rc = zalloc(sim, (size_t)d.E, &d.reb_list)) ||
        (rc = zalloc(sim, 1, &d.nreb)) ||
        (rc = zalloc(sim, 1, &sim->d_flag)) || (rc = zalloc(sim, 1, &sim->d_loop)) || (rc = zalloc(sim, (size_t)d.kmax, &sim->d_dbg_cand)) ||
        (rc = zalloc(sim, 1, &sim->d_dbg_cnt)) || (rc = zalloc(sim, 3 * (size_t)nv, &sim->d_scratch)))
      goto fail;
    if (cudaMallocHost(&sim->h_flag, sizeof(int)) != cudaSuccess) { rc = TAC_ENOMEM; goto fail; }
    if ((rc = upload_env_material(sim, 0))) { sim->err = "upload per-env material"; goto fail; }
    int prio_lo = 0, prio_hi = 0;  // the rebuild's few long warps must start before the element pass fills the SMs
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&d.side, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&d.side2, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&d.side3, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&d.side4, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_join4, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_reb, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&sim->cap, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_cls, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_join2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_join, cudaEventDisableTiming) != cudaSuccess) {
      rc = TAC_ECUDA; sim->err = "side stream / events"; goto fail;
    }
    // initial poses: per-env fp64 state on the host, then upload
    std::vector<EnvS> es(d.E);
    for (int e = 0; e < d.E; ++e) {
      memset(&es[e], 0, sizeof(EnvS));
      const float* q = info->init_poses + 7 * e;
      double w = q[3], x = q[4], y = q[5], z = q[6];
      double n = std::sqrt(w * w + x * x + y * y + z * z);
      if (!(n > 0)) { rc = TAC_EINVAL; sim->err = "zero quaternion in init_poses"; goto fail; }
      w /= n; x /= n; y /= n; z /= n;
      double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                     2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                     2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
      for (int i = 0; i < 3; ++i) es[e].c[i] = es[e].ct[i] = es[e].cs[i] = q[i];
      for (int i = 0; i < 9; ++i) es[e].R[i] = es[e].Rt[i] = es[e].Rs[i] = R[i];
      es[e].mode = kActive;
    }
    if (cudaMemcpy(d.es, es.data(), sizeof(EnvS) * d.E, cudaMemcpyHostToDevice) != cudaSuccess) {
      rc = TAC_ECUDA; sim->err = "upload env state"; goto fail;
    }
    // feasibility of the initial poses: no candidate within dhat may have d <= 0
    launch_broadphase(d, false, 0);
    std::vector<int> run(d.Es, 1);
    if (cudaMemcpy(d.run, run.data(), sizeof(int) * d.Es, cudaMemcpyHostToDevice) != cudaSuccess) { rc = TAC_ECUDA; goto fail; }
    cudaMemset(d.nreb, 0, sizeof(int));
    launch_eval(d, 1e-3, 0);  // energies at rest: infinite barrier energy <=> touching / intersecting
    if (cudaDeviceSynchronize() != cudaSuccess) { rc = TAC_ECUDA; sim->err = "initial feasibility check failed"; goto fail; }
    std::vector<EnvS> chk(d.E);
    cudaMemcpy(chk.data(), d.es, sizeof(EnvS) * d.E, cudaMemcpyDeviceToHost);
    for (int e = 0; e < d.E; ++e)
      if (chk[e].flags & 8) { rc = TAC_EINVAL; sim->err = "indenter touches the gel at its initial pose (env " + std::to_string(e) + ")"; goto fail; }
    {  // deep intersections: a gel surface edge crossing an indenter triangle
      int* dhit = nullptr;
      std::vector<int> hit(d.E, 0);
      if (cudaMalloc(&dhit, sizeof(int) * d.E) != cudaSuccess) { rc = TAC_ENOMEM; goto fail; }
      cudaMemset(dhit, 0, sizeof(int) * d.E);
      launch_intersect_check(d, dhit, 0);
      cudaError_t ce = cudaMemcpy(hit.data(), dhit, sizeof(int) * d.E, cudaMemcpyDeviceToHost);
      cudaFree(dhit);
      if (ce != cudaSuccess) { rc = TAC_ECUDA; sim->err = "initial intersection check failed"; goto fail; }
      for (int e = 0; e < d.E; ++e)
        if (hit[e]) { rc = TAC_EINVAL; sim->err = "indenter intersects the gel at its initial pose (env " + std::to_string(e) + ")"; goto fail; }
    }
    // restore the clean initial state
    if (cudaMemcpy(d.es, es.data(), sizeof(EnvS) * d.E, cudaMemcpyHostToDevice) != cudaSuccess) { rc = TAC_ECUDA; goto fail; }
    cudaMemset(d.acc, 0, sizeof(double) * kNAcc * d.Es);
    cudaMemset(d.run, 0, sizeof(int) * d.Es);
    cudaMemset(d.ncand, 0, sizeof(int) * 2 * d.E);
    cudaMemset(d.u, 0, sizeof(float) * nvec);
    cudaMemset(d.g, 0, sizeof(float) * nvec);
    cudaMemset(d.D, 0, sizeof(float) * 2 * nvec);
    if (cudaDeviceSynchronize() != cudaSuccess) { rc = TAC_ECUDA; goto fail; }
  }
  *out = sim;
  return TAC_OK;
fail:
  g_create_err = sim->err.empty() ? "tac_create failed" : sim->err;
  tac_destroy(sim);
  return rc ? rc : TAC_ECUDA;
}

tac_status tac_destroy(tac_sim* sim) {
  if (!sim) return TAC_OK;
  cudaSetDevice(sim->device);
  if (sim->d.side) { cudaStreamSynchronize(sim->d.side); cudaStreamDestroy(sim->d.side); }
  if (sim->d.side2) { cudaStreamSynchronize(sim->d.side2); cudaStreamDestroy(sim->d.side2); }
  if (sim->d.side3) { cudaStreamSynchronize(sim->d.side3); cudaStreamDestroy(sim->d.side3); }
  if (sim->d.side4) { cudaStreamSynchronize(sim->d.side4); cudaStreamDestroy(sim->d.side4); }
  for (auto& g : sim->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& g : sim->wgraphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (sim->cap) cudaStreamDestroy(sim->cap);
  for (cudaEvent_t ev : {sim->d.ev_fork, sim->d.ev_join, sim->d.ev_cls, sim->d.ev_join2, sim->d.ev_reb, sim->d.ev_join4})
    if (ev) cudaEventDestroy(ev);
  for (void* p : sim->allocs) cudaFree(p);
  if (sim->h_flag) cudaFreeHost(sim->h_flag);
  delete sim->prof;
  delete sim;
  return TAC_OK;
}

static tac_status check_sim(tac_sim* sim) {
  if (!sim) return TAC_EINVAL;
  if (sim->sticky) return TAC_ECUDA;
  return TAC_OK;
}
static tac_status post_launch(tac_sim* sim) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    sim->err = std::string("kernel launch: ") + cudaGetErrorString(e);
    sim->sticky = true;
    return TAC_ECUDA;
  }
  return TAC_OK;
}

// n PNCG iterations; with `fin` the last one is the step's final evaluation: Armijo and
// the convergence test only (the step then commits the last accepted iterate, R31)
static void launch_iterations(const Dev& d, double h, int n, bool fin, cudaStream_t s) {
  for (int it = 0; it < n; ++it) {
    const bool tl = it == g_tl_iter;
    if (tl) {
      cudaEventCreate(&g_tl.start);
      cudaEventRecord(g_tl.start, s);
      g_tl_on = true;
    }
    launch_eval(d, h, s);       // a4 + a5 + Armijo (a8)
    if (fin && it == n - 1) {
      launch_direction(d, s, false);  // a8 convergence test
      if (g_prof == nullptr) cudaStreamWaitEvent(s, d.ev_reb, 0);  // join the pipelined rebuild (R16)
      break;
    }
    launch_direction(d, s);     // a6
    launch_curvature(d, h, s);  // a7
    launch_alpha(d, h, s);      // a7/a8 (+ a2 rebuild)
    if (tl) {
      g_tl_on = false;
      tl_print();
    }
  }
}

// n PNCG iterations on stream s (the last one the step's final evaluation if `fin`):
// replayed from a cached CUDA graph unless per-launch profiling is on (its events sit
// between the launches) or graphs are disabled.  Graphs are keyed by (anchor buffer, h, n,
// fin): the fixed mode uses one per anchor buffer, the tolerance mode a chunk graph and a
// final-chunk graph per anchor buffer.
static bool run_iterations(tac_sim* sim, double h, int n, bool fin, cudaStream_t s) {
  const Dev& d = sim->d;
  if (sim->prof || !sim->use_graphs) {
    launch_iterations(d, h, n, fin, s);
    return true;
  }
  tac_sim::IterGraph* G = nullptr;
  for (auto& g : sim->graphs)
    if (g.exec && g.anc == (const void*)d.anc && g.h == h && g.n == n && g.fin == fin) G = &g;
  if (!G) {  // capture into an empty slot, else the least recently used one
    G = &sim->graphs[0];
    for (auto& g : sim->graphs) {
      if (!g.exec) { G = &g; break; }
      if (g.used < G->used) G = &g;
    }
    if (G->exec) { cudaGraphExecDestroy(G->exec); G->exec = nullptr; }
    const long long l0 = g_launches;
    cudaGraph_t gr = nullptr;
    bool ok = cudaStreamBeginCapture(sim->cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      launch_iterations(d, h, n, fin, sim->cap);
      ok = cudaStreamEndCapture(sim->cap, &gr) == cudaSuccess && gr;
    }
    // kernel nodes keep their stream's priority (the contact chain's high priority)
    ok = ok && cudaGraphInstantiateWithFlags(&G->exec, gr, cudaGraphInstantiateFlagUseNodePriority) == cudaSuccess;
    if (gr) cudaGraphDestroy(gr);
    if (!ok) {  // capture unsupported here: launch the same kernels directly from now on
      cudaGetLastError();
      if (G->exec) cudaGraphExecDestroy(G->exec);
      *G = tac_sim::IterGraph{};
      sim->use_graphs = false;
      g_launches = l0;
      if (getenv("TAC_GRAPH_DEBUG")) fprintf(stderr, "tac: iteration graph capture failed, direct launches\n");
      launch_iterations(d, h, n, fin, s);
      return true;
    }
    G->anc = d.anc;
    G->h = h;
    G->n = n;
    G->fin = fin;
    G->launches = g_launches - l0;
    g_launches = l0;
  }
  G->used = ++sim->graph_clock;
  g_launches += G->launches;
  return cudaGraphLaunch(G->exec, s) == cudaSuccess;
}

// Tolerance mode's iteration loop on the device: a graph whose WHILE node runs (one PNCG
// iteration + k_loop_ctl) until no env is active or K - 1 iterations have run.  Returns
// false if conditional graphs are unavailable (the caller falls back to host-polled chunks).
static bool run_while_loop(tac_sim* sim, double h, int K, cudaStream_t s) {
  const Dev& d = sim->d;
  tac_sim::WhileGraph* G = nullptr;
  for (auto& g : sim->wgraphs)
    if (g.exec && g.anc == (const void*)d.anc && g.h == h && g.K == K) G = &g;
  if (!G) {
    G = &sim->wgraphs[0];
    for (auto& g : sim->wgraphs)
      if (g.anc == (const void*)d.anc || !g.exec) { G = &g; break; }
    if (G->exec) { cudaGraphExecDestroy(G->exec); G->exec = nullptr; }
    cudaGraph_t gr = nullptr;
    bool ok = cudaGraphCreate(&gr, 0) == cudaSuccess;
    cudaGraphConditionalHandle hnd;
    ok = ok && cudaGraphConditionalHandleCreate(&hnd, gr, 1, cudaGraphCondAssignDefault) == cudaSuccess;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hnd;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    ok = ok && cudaGraphAddNode(&node, gr, nullptr, 0, &cp) == cudaSuccess;
    const long long l0 = g_launches;
    if (ok) {
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      ok = cudaStreamBeginCaptureToGraph(sim->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
           cudaSuccess;
      if (ok) {
        // loop control in k_alpha's last block (one launch per trip less than a k_loop_ctl;
        // TAC_LOOP_CTL_KERNEL=1 keeps the separate kernel for A/B)
        Dev dl = d;
        const bool sep = getenv("TAC_LOOP_CTL_KERNEL") != nullptr;
        if (!sep) { dl.loop_on = 1; dl.loop_h = hnd; dl.loop_ctr = sim->d_loop; dl.loop_limit = K - 1; }
        launch_iterations(dl, h, 1, false, sim->cap);
        if (sep) launch_loop_ctl(d, hnd, sim->d_loop, K - 1, sim->cap);
        cudaGraph_t out = nullptr;
        ok = cudaStreamEndCapture(sim->cap, &out) == cudaSuccess;
      }
    }
    ok = ok && cudaGraphInstantiateWithFlags(&G->exec, gr, cudaGraphInstantiateFlagUseNodePriority) == cudaSuccess;
    if (gr) cudaGraphDestroy(gr);
    G->launches_per_trip = g_launches - l0;
    g_launches = l0;
    if (!ok) {
      cudaGetLastError();
      if (G->exec) cudaGraphExecDestroy(G->exec);
      *G = tac_sim::WhileGraph{};
      sim->use_while = false;
      if (getenv("TAC_GRAPH_DEBUG")) fprintf(stderr, "tac: WHILE-node graph unavailable, host-polled chunks\n");
      return false;
    }
    G->anc = d.anc;
    G->h = h;
    G->K = K;
  }
  sim->while_per_trip = G->launches_per_trip;  // the trip count is only known on the device
  if (cudaMemsetAsync(sim->d_loop, 0, sizeof(int), s) != cudaSuccess) return false;
  return cudaGraphLaunch(G->exec, s) == cudaSuccess;
}

tac_status tac_step(tac_sim* sim, const float* target_poses, float dt, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!target_poses || !(dt > 0)) { sim->err = "tac_step: null poses or dt <= 0"; return TAC_EINVAL; }
  cudaSetDevice(sim->device);
  cudaStream_t s = (cudaStream_t)stream;
  const Dev& d = sim->d;
  double h = dt;
  g_launches = 0;
  sim->while_per_trip = 0;
  g_prof = sim->prof;
  launch_step_setup(d, target_poses, h, sim->step_count++, s);  // a1
  cudaMemsetAsync(d.nreb, 0, sizeof(int), s);  // rebuilds flagged by the last step's final alpha are superseded
  launch_broadphase(d, false, s);            // a2
  launch_anchors(d, h, s);                   // a3
  launch_sort_anchors(d, sim->d.anc2, s);    // neighbouring anchors share gel corners (friction scatter)
  std::swap(sim->d.anc, sim->d.anc2);        // launches below read the sorted buffer
  int K = sim->fixed_iters > 0 ? sim->fixed_iters : sim->max_iters;
  if (sim->fixed_iters == 0 && K > 1 && sim->use_while && sim->use_graphs && !sim->prof) {
    // tolerance mode: K - 1 iterations under device-side control, then the final evaluation
    if (run_while_loop(sim, h, K, s)) {
      if (!run_iterations(sim, h, 1, true, s)) { g_prof = nullptr; return post_launch(sim); }
      launch_finalize(d, h, s);  // a9
      sim->launches = g_launches;
      g_prof = nullptr;
      return post_launch(sim);
    }
  }
  const int chunk = sim->fixed_iters > 0 ? K : std::min(K, sim->check_every);
  for (int it = 0; it < K;) {
    const int n = std::min(chunk, K - it);
    if (!run_iterations(sim, h, n, it + n == K, s)) { g_prof = nullptr; return post_launch(sim); }
    it += n;
    if (sim->fixed_iters == 0 && it % sim->check_every == 0 && it < K) {  // all envs done?
      cudaMemsetAsync(sim->d_flag, 0, sizeof(int), s);
      launch_any_active(d, sim->d_flag, s);
      cudaMemcpyAsync(sim->h_flag, sim->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) { g_prof = nullptr; return post_launch(sim); }
      if (*sim->h_flag == 0) break;
    }
  }
  launch_finalize(d, h, s);  // a9
  sim->launches = g_launches;
  g_prof = nullptr;
  return post_launch(sim);
}

tac_status tac_markers(tac_sim* sim, float* out, int32_t ncomp, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!out || (ncomp != 2 && ncomp != 3)) { sim->err = "tac_markers: bad output or ncomp"; return TAC_EINVAL; }
  cudaSetDevice(sim->device);
  g_launches = 0;
  g_prof = sim->prof;
  launch_markers(sim->d, out, ncomp, (cudaStream_t)stream);
  g_prof = nullptr;
  sim->launches = g_launches;
  sim->while_per_trip = 0;  // this call's launches only
  return post_launch(sim);
}

// ------------------------------------------------------------ marker all-gather over NCCL
// NCCL entry points resolved at run time (no link dependency; the process's already-loaded
// libnccl.so.2 -- torch's -- is preferred so one NCCL serves the whole process).
namespace {
typedef struct { char internal[128]; } nccl_uid;
typedef int (*nccl_get_uid_t)(nccl_uid*);
typedef int (*nccl_init_rank_t)(void**, int, nccl_uid, int);
typedef int (*nccl_destroy_t)(void*);
typedef int (*nccl_allgather_t)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*nccl_user_rank_t)(const void*, int*);
typedef int (*nccl_count_t)(const void*, int*);
typedef const char* (*nccl_errstr_t)(int);
struct NcclApi {
  bool ok = false;
  nccl_get_uid_t get_uid = nullptr;
  nccl_init_rank_t init_rank = nullptr;
  nccl_destroy_t destroy = nullptr;
  nccl_allgather_t allgather = nullptr;
  nccl_user_rank_t user_rank = nullptr;
  nccl_count_t count = nullptr;
  nccl_errstr_t errstr = nullptr;
};
constexpr int kNcclFloat32 = 7;  // ncclFloat32 in nccl.h's ncclDataType_t
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return a;
    a.get_uid = (nccl_get_uid_t)dlsym(h, "ncclGetUniqueId");
    a.init_rank = (nccl_init_rank_t)dlsym(h, "ncclCommInitRank");
    a.destroy = (nccl_destroy_t)dlsym(h, "ncclCommDestroy");
    a.allgather = (nccl_allgather_t)dlsym(h, "ncclAllGather");
    a.user_rank = (nccl_user_rank_t)dlsym(h, "ncclCommUserRank");
    a.count = (nccl_count_t)dlsym(h, "ncclCommCount");
    a.errstr = (nccl_errstr_t)dlsym(h, "ncclGetErrorString");
    a.ok = a.get_uid && a.init_rank && a.destroy && a.allgather && a.user_rank && a.count && a.errstr;
    return a;
  }();
  return api;
}
}  // namespace

tac_status tac_nccl_unique_id(uint8_t out[128]) {
  if (!out || !nccl().ok) return TAC_EINVAL;
  nccl_uid id;
  if (nccl().get_uid(&id) != 0) return TAC_ECUDA;
  std::memcpy(out, id.internal, 128);
  return TAC_OK;
}

tac_status tac_nccl_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks || !nccl().ok) return TAC_EINVAL;
  *comm = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return TAC_ECUDA;
  nccl_uid u;
  std::memcpy(u.internal, id, 128);
  return nccl().init_rank(comm, nranks, u, rank) == 0 ? TAC_OK : TAC_ECUDA;
}

tac_status tac_nccl_comm_destroy(void* comm) {
  if (!comm || !nccl().ok) return TAC_EINVAL;
  return nccl().destroy(comm) == 0 ? TAC_OK : TAC_ECUDA;
}

tac_status tac_gather_markers(tac_sim* sim, void* comm, float* recvbuf, int32_t ncomp, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!comm || !recvbuf || (ncomp != 2 && ncomp != 3)) { sim->err = "tac_gather_markers: bad argument"; return TAC_EINVAL; }
  if (!nccl().ok) { sim->err = "tac_gather_markers: NCCL not available"; return TAC_EINVAL; }
  int rank = 0, nranks = 0;
  if (nccl().user_rank(comm, &rank) != 0 || nccl().count(comm, &nranks) != 0) {
    sim->err = "tac_gather_markers: invalid communicator";
    return TAC_EINVAL;
  }
  cudaSetDevice(sim->device);
  const size_t count = (size_t)sim->d.E * sim->d.nm * ncomp;
  float* slot = recvbuf + (size_t)rank * count;
  g_launches = 0;
  g_prof = sim->prof;
  launch_markers(sim->d, slot, ncomp, (cudaStream_t)stream);  // this rank's slot, then in place
  g_prof = nullptr;
  sim->launches = g_launches;
  sim->while_per_trip = 0;
  if ((st = post_launch(sim))) return st;
  const int rc = nccl().allgather(slot, recvbuf, count, kNcclFloat32, comm, (cudaStream_t)stream);
  if (rc != 0) {
    sim->err = std::string("ncclAllGather: ") + nccl().errstr(rc);
    return TAC_ECUDA;
  }
  return TAC_OK;
}

tac_status tac_marker_sqerr(tac_sim* sim, const float* ref, double* acc, int32_t ncomp, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!ref || !acc || (ncomp != 2 && ncomp != 3)) { sim->err = "tac_marker_sqerr: bad pointer or ncomp"; return TAC_EINVAL; }
  cudaSetDevice(sim->device);
  g_launches = 0;
  g_prof = sim->prof;
  launch_marker_sqerr(sim->d, ref, acc, ncomp, (cudaStream_t)stream);
  g_prof = nullptr;
  sim->launches = g_launches;
  sim->while_per_trip = 0;  // this call's launches only
  return post_launch(sim);
}

// ------------------------------------------------------------ checkpoint / resume
// layout: 64-byte header {magic, version, nv, Es, E, sizeof(EnvS), step_count}, u^t, v^t
// ([3][nv][Es] fp32 each, the AoSoA layout), EnvS [E]
namespace {
constexpr uint64_t kCkptMagic = 0x54414331434b5054ull;  // "TPKC1CAT"
struct CkptHeader {
  uint64_t magic, version, nv, Es, E, envs_bytes, step_count, pad;
};
static_assert(sizeof(CkptHeader) == 64, "checkpoint header");
size_t ckpt_vec_bytes(const Dev& d) { return sizeof(float) * 3 * (size_t)d.nv * d.Es; }
size_t ckpt_bytes(const Dev& d) { return sizeof(CkptHeader) + 2 * ckpt_vec_bytes(d) + sizeof(EnvS) * (size_t)d.E; }
}  // namespace

tac_status tac_checkpoint_size(const tac_sim* sim, uint64_t* bytes) {
  if (!sim || !bytes) return TAC_EINVAL;
  *bytes = ckpt_bytes(sim->d);
  return TAC_OK;
}

tac_status tac_checkpoint_save(tac_sim* sim, void* dst, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!dst) { sim->err = "tac_checkpoint_save: null buffer"; return TAC_EINVAL; }
  cudaSetDevice(sim->device);
  const Dev& d = sim->d;
  cudaStream_t s = (cudaStream_t)stream;
  CkptHeader h{kCkptMagic, 1, (uint64_t)d.nv, (uint64_t)d.Es, (uint64_t)d.E, sizeof(EnvS) * (uint64_t)d.E,
               sim->step_count, 0};
  char* p = (char*)dst;
  // the header travels as a kernel argument (captured at launch: no host buffer to keep alive)
  launch_write_words(d, (uint64_t*)p, (const uint64_t*)&h, sizeof(h) / 8, s);
  p += sizeof(h);
  CK(cudaMemcpyAsync(p, d.ut, ckpt_vec_bytes(d), cudaMemcpyDeviceToDevice, s));
  p += ckpt_vec_bytes(d);
  CK(cudaMemcpyAsync(p, d.vt, ckpt_vec_bytes(d), cudaMemcpyDeviceToDevice, s));
  p += ckpt_vec_bytes(d);
  CK(cudaMemcpyAsync(p, d.es, sizeof(EnvS) * (size_t)d.E, cudaMemcpyDeviceToDevice, s));
  return post_launch(sim);
}

tac_status tac_checkpoint_load(tac_sim* sim, const void* src, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!src) { sim->err = "tac_checkpoint_load: null buffer"; return TAC_EINVAL; }
  cudaSetDevice(sim->device);
  const Dev& d = sim->d;
  cudaStream_t s = (cudaStream_t)stream;
  CkptHeader h;
  CK(cudaMemcpyAsync(&h, src, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h.magic != kCkptMagic || h.version != 1 || h.nv != (uint64_t)d.nv || h.Es != (uint64_t)d.Es ||
      h.E != (uint64_t)d.E || h.envs_bytes != sizeof(EnvS) * (uint64_t)d.E) {
    sim->err = "tac_checkpoint_load: not a checkpoint of a simulator of this size";
    return TAC_EINVAL;
  }
  const char* p = (const char*)src + sizeof(h);
  CK(cudaMemcpyAsync(d.ut, p, ckpt_vec_bytes(d), cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(d.u, p, ckpt_vec_bytes(d), cudaMemcpyDeviceToDevice, s));
  p += ckpt_vec_bytes(d);
  CK(cudaMemcpyAsync(d.vt, p, ckpt_vec_bytes(d), cudaMemcpyDeviceToDevice, s));
  p += ckpt_vec_bytes(d);
  CK(cudaMemcpyAsync(d.es, p, sizeof(EnvS) * (size_t)d.E, cudaMemcpyDeviceToDevice, s));
  sim->step_count = h.step_count;
  return TAC_OK;
}

tac_status tac_reset(tac_sim* sim, const uint8_t* env_mask, const float* poses, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!env_mask || !poses) { sim->err = "tac_reset: null pointer"; return TAC_EINVAL; }
  cudaSetDevice(sim->device);
  launch_reset(sim->d, env_mask, poses, (cudaStream_t)stream);
  return post_launch(sim);
}

tac_status tac_set_env_material(tac_sim* sim, const double* E, const double* nu, const double* rho,
                                const double* mu_f, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  const int n = sim->d.E;
  for (int e = 0; e < n; ++e) {  // validate everything before changing anything
    if ((E && !(E[e] > 0)) || (nu && !(nu[e] >= 0 && nu[e] < 0.5)) || (rho && !(rho[e] > 0)) ||
        (mu_f && !(mu_f[e] >= 0))) {
      sim->err = "tac_set_env_material: invalid material for env " + std::to_string(e);
      return TAC_EINVAL;
    }
  }
  for (int e = 0; e < n; ++e) {
    if (E) sim->thE[e] = E[e];
    if (nu) sim->thNu[e] = nu[e];
    if (rho) sim->thRho[e] = rho[e];
    if (mu_f) sim->thMu[e] = mu_f[e];
  }
  cudaSetDevice(sim->device);
  if ((st = upload_env_material(sim, (cudaStream_t)stream))) { sim->err = "tac_set_env_material: upload failed"; return st; }
  return TAC_OK;
}

tac_status tac_set_pose_noise(tac_sim* sim, double sigma_t, double sigma_r, uint64_t seed, int64_t env_offset) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!(sigma_t >= 0) || !(sigma_r >= 0) || env_offset < 0) { sim->err = "tac_set_pose_noise: bad arguments"; return TAC_EINVAL; }
  sim->d.noise_t = sigma_t;
  sim->d.noise_r = sigma_r;
  sim->d.noise_seed = seed;
  sim->d.env_offset = env_offset;
  return TAC_OK;
}

tac_status tac_env_status(tac_sim* sim, int32_t* iters, float* pg_norm, uint32_t* flags, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  cudaSetDevice(sim->device);
  launch_status(sim->d, iters, pg_norm, flags, (cudaStream_t)stream);
  return post_launch(sim);
}

tac_status tac_info(const tac_sim* sim, int32_t* out) {
  if (!sim || !out) return TAC_EINVAL;
  const Dev& d = sim->d;
  int v[10] = {d.nv, d.nt, d.E, d.Es, d.nm, d.nsv, d.nse, d.nst, d.ncells, d.nrest};
  memcpy(out, v, sizeof(v));
  return TAC_OK;
}

int64_t tac_last_launch_count(const tac_sim* sim) {
  if (!sim) return 0;
  if (sim->while_per_trip == 0) return sim->launches;
  // tolerance mode's device-side loop: its trip count is read back (synchronises the device)
  int trips = 0;
  cudaSetDevice(sim->device);
  if (cudaMemcpy(&trips, sim->d_loop, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return sim->launches;
  return sim->launches + (long long)trips * sim->while_per_trip;
}

tac_status tac_profile_enable(tac_sim* sim, int32_t on) {
  if (!sim) return TAC_EINVAL;
  cudaSetDevice(sim->device);
  if (on && !sim->prof) sim->prof = new tac::Profiler;
  if (!on && sim->prof) { delete sim->prof; sim->prof = nullptr; }
  return TAC_OK;
}

tac_status tac_profile_read(tac_sim* sim, double* ms, int64_t* counts, int32_t n) {
  if (!sim || !sim->prof) return TAC_ESTATE;
  cudaSetDevice(sim->device);
  sim->prof->drain();
  for (int k = 0; k < n && k < KID_COUNT; ++k) {
    if (ms) ms[k] = sim->prof->ms[k];
    if (counts) counts[k] = sim->prof->cnt[k];
    sim->prof->ms[k] = 0;
    sim->prof->cnt[k] = 0;
  }
  return TAC_OK;
}

const char* tac_profile_kernel_name(int32_t id) { return tac::kernel_name(id); }

tac_status tac_env_stats(tac_sim* sim, int32_t* out, void* stream) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (!out) return TAC_EINVAL;
  cudaSetDevice(sim->device);
  launch_stats(sim->d, (int4*)out, (cudaStream_t)stream);
  return post_launch(sim);
}

// ---------------------------------------------------------------- debug hooks
// host <-> device copies of one env's vertex vector in the AoSoA layout [v][Es/32][c][32]
static tac_status copy_env_comp(tac_sim* sim, float* host, const float* dev_base, int env, int c, int ncomp,
                                bool to_host) {
  const Dev& d = sim->d;
  size_t pitch = sizeof(float) * (size_t)(d.Es / 32) * ncomp * 32;
  size_t off = ((size_t)(env / 32) * ncomp + c) * 32 + (env % 32);
  if (to_host)
    CK(cudaMemcpy2D(host, sizeof(float), dev_base + off, pitch, sizeof(float), d.nv, cudaMemcpyDeviceToHost));
  else
    CK(cudaMemcpy2D((float*)dev_base + off, pitch, host, sizeof(float), sizeof(float), d.nv, cudaMemcpyHostToDevice));
  return TAC_OK;
}
static tac_status gather_vec(tac_sim* sim, const float* dsrc, int env, double* out) {
  const Dev& d = sim->d;
  std::vector<float> tmp((size_t)d.nv);
  for (int c = 0; c < 3; ++c) {
    tac_status st = copy_env_comp(sim, tmp.data(), dsrc, env, c, 3, true);
    if (st) return st;
    for (int v = 0; v < d.nv; ++v) out[3 * v + c] = tmp[v];
  }
  return TAC_OK;
}
static tac_status scatter_vec(tac_sim* sim, float* ddst, int env, const double* in) {
  const Dev& d = sim->d;
  std::vector<float> tmp((size_t)d.nv);
  for (int c = 0; c < 3; ++c) {
    for (int v = 0; v < d.nv; ++v) tmp[v] = (float)in[3 * v + c];
    tac_status st = copy_env_comp(sim, tmp.data(), ddst, env, c, 3, false);
    if (st) return st;
  }
  return TAC_OK;
}

tac_status tac_get_state(tac_sim* sim, int32_t env, double* u, double* v, double* c, double* R) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (env < 0 || env >= sim->d.E) return TAC_EINVAL;
  cudaSetDevice(sim->device);
  CK(cudaDeviceSynchronize());
  if (u && (st = gather_vec(sim, sim->d.ut, env, u))) return st;
  if (v && (st = gather_vec(sim, sim->d.vt, env, v))) return st;
  EnvS es;
  CK(cudaMemcpy(&es, sim->d.es + env, sizeof(EnvS), cudaMemcpyDeviceToHost));
  if (c) for (int i = 0; i < 3; ++i) c[i] = es.ct[i];
  if (R) for (int i = 0; i < 9; ++i) R[i] = es.Rt[i];
  return TAC_OK;
}

tac_status tac_set_state(tac_sim* sim, int32_t env, const double* u, const double* v, const double* c,
                         const double* R) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (env < 0 || env >= sim->d.E || !u || !v || !c || !R) return TAC_EINVAL;
  cudaSetDevice(sim->device);
  CK(cudaDeviceSynchronize());
  if ((st = scatter_vec(sim, sim->d.ut, env, u)) || (st = scatter_vec(sim, sim->d.u, env, u)) ||
      (st = scatter_vec(sim, sim->d.vt, env, v)))
    return st;
  EnvS es;
  CK(cudaMemcpy(&es, sim->d.es + env, sizeof(EnvS), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 3; ++i) es.c[i] = es.ct[i] = c[i];
  for (int i = 0; i < 9; ++i) es.R[i] = es.Rt[i] = R[i];
  CK(cudaMemcpy(sim->d.es + env, &es, sizeof(EnvS), cudaMemcpyHostToDevice));
  return TAC_OK;
}

tac_status tac_debug_surface(const tac_sim* sim, int32_t* sv, int32_t* se, int32_t* st, int32_t* ie, int32_t* counts) {
  if (!sim) return TAC_EINVAL;
  if (sv) memcpy(sv, sim->sv.data(), sizeof(int) * sim->sv.size());
  if (se) memcpy(se, sim->se_flat.data(), sizeof(int) * sim->se_flat.size());
  if (st) memcpy(st, sim->st_flat.data(), sizeof(int) * sim->st_flat.size());
  if (ie) memcpy(ie, sim->ie_flat.data(), sizeof(int) * sim->ie_flat.size());
  if (counts) counts[0] = (int)sim->ie_flat.size() / 2;
  return TAC_OK;
}

tac_status tac_debug_marker_map(const tac_sim* sim, int32_t* tet, int32_t* idx, double* w) {
  if (!sim) return TAC_EINVAL;
  int nm = sim->d.nm;
  if (tet) memcpy(tet, sim->mk_tet.data(), sizeof(int) * nm);
  if (idx) memcpy(idx, sim->mk_idx.data(), sizeof(int) * 4 * nm);
  if (w) memcpy(w, sim->mk_w.data(), sizeof(double) * 4 * nm);
  return TAC_OK;
}

static tac_status set_pose_current(tac_sim* sim, int env, const double* c, const double* R) {
  EnvS es;
  CK(cudaMemcpy(&es, sim->d.es + env, sizeof(EnvS), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 3; ++i) es.c[i] = c[i];
  for (int i = 0; i < 9; ++i) es.R[i] = R[i];
  es.mode = kActive;
  CK(cudaMemcpy(sim->d.es + env, &es, sizeof(EnvS), cudaMemcpyHostToDevice));
  return TAC_OK;
}

tac_status tac_debug_broadphase(tac_sim* sim, int32_t env, const float* u, const double* c, const double* R,
                                double r, int32_t* out, int32_t cap, int32_t* n) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (env < 0 || env >= sim->d.E || !u || !c || !R || !n) return TAC_EINVAL;
  cudaSetDevice(sim->device);
  Dev d = sim->d;
  std::vector<double> ud(3 * (size_t)d.nv);
  for (size_t i = 0; i < ud.size(); ++i) ud[i] = u[i];
  if ((st = scatter_vec(sim, d.u, env, ud.data())) || (st = set_pose_current(sim, env, c, R))) return st;
  // run the production kernel restricted to this env (E = env + 1, blocks of env only)
  CK(cudaMemset(sim->d_dbg_cnt, 0, sizeof(int)));
  Dev dd = d;
  dd.E = env + 1;
  std::vector<EnvS> all(env + 1);
  CK(cudaMemcpy(all.data(), d.es, sizeof(EnvS) * (env + 1), cudaMemcpyDeviceToHost));
  std::vector<EnvS> masked = all;
  for (int e = 0; e < env; ++e) masked[e].mode = kDone;
  CK(cudaMemcpy(d.es, masked.data(), sizeof(EnvS) * (env + 1), cudaMemcpyHostToDevice));
  launch_debug_broadphase(dd, r, sim->d_dbg_cand, sim->d_dbg_cnt, d.kmax, 0);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(d.es, all.data(), sizeof(EnvS) * (env + 1), cudaMemcpyHostToDevice));
  int cnt = 0;
  CK(cudaMemcpy(&cnt, sim->d_dbg_cnt, sizeof(int), cudaMemcpyDeviceToHost));
  *n = cnt;
  int m = std::min(std::min(cnt, cap), d.kmax);
  std::vector<unsigned long long> rec(m);
  if (m) CK(cudaMemcpy(rec.data(), sim->d_dbg_cand, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost));
  for (int i = 0; i < m; ++i) {
    out[3 * i] = (int)(rec[i] >> 62);
    out[3 * i + 1] = (int)((rec[i] >> 31) & 0x7fffffffu);
    out[3 * i + 2] = (int)(rec[i] & 0x7fffffffu);
  }
  return post_launch(sim);
}

tac_status tac_debug_eval(tac_sim* sim, int32_t env, const double* u_t, const double* v_t, const double* c_t,
                          const double* R_t, const double* u, const double* c, const double* R,
                          const double* target7, double dt, double* parts, double* g, double* D, double* grig,
                          double* Drig) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (env < 0 || env >= sim->d.E || !(dt > 0)) return TAC_EINVAL;
  cudaSetDevice(sim->device);
  Dev d = sim->d;
  if ((st = tac_set_state(sim, env, u_t, v_t, c_t, R_t))) return st;
  // step setup for all envs with the target, then mask every other env
  std::vector<float> poses(7 * (size_t)d.E, 0.f);
  std::vector<EnvS> all(d.E);
  CK(cudaMemcpy(all.data(), d.es, sizeof(EnvS) * d.E, cudaMemcpyDeviceToHost));
  for (int e = 0; e < d.E; ++e) {
    for (int i = 0; i < 3; ++i) poses[7 * e + i] = (float)all[e].ct[i];
    poses[7 * e + 3] = 1.f;
  }
  for (int i = 0; i < 7; ++i) poses[7 * env + i] = (float)target7[i];
  float* dp = nullptr;
  CK(cudaMalloc(&dp, sizeof(float) * poses.size()));
  CK(cudaMemcpy(dp, poses.data(), sizeof(float) * poses.size(), cudaMemcpyHostToDevice));
  launch_step_setup(d, dp, dt, 0ull, 0);
  CK(cudaDeviceSynchronize());
  cudaFree(dp);
  std::vector<EnvS> es(d.E);
  CK(cudaMemcpy(es.data(), d.es, sizeof(EnvS) * d.E, cudaMemcpyDeviceToHost));
  for (int e = 0; e < d.E; ++e)
    if (e != env) es[e].mode = kDone;
  CK(cudaMemcpy(d.es, es.data(), sizeof(EnvS) * d.E, cudaMemcpyHostToDevice));
  std::vector<int> run(d.Es, 0);
  run[env] = 1;
  CK(cudaMemcpy(d.run, run.data(), sizeof(int) * d.Es, cudaMemcpyHostToDevice));
  launch_broadphase(d, false, 0);
  launch_anchors(d, dt, 0);
  // move to the evaluation state (u, c, R) and rebuild the candidates there
  if ((st = scatter_vec(sim, d.u, env, u)) || (st = set_pose_current(sim, env, c, R))) return st;
  CK(cudaMemset(d.lbuf + env, 0, sizeof(int)));  // active buffer 0
  CK(cudaMemset(d.ncand + env, 0, sizeof(int)));
  launch_broadphase(d, false, 0);
  CK(cudaMemset(d.nreb, 0, sizeof(int)));
  launch_eval(d, dt, 0);
  CK(cudaDeviceSynchronize());
  // results: accept kernel stored the energy and rigid terms in EnvS; g / D in the vectors
  EnvS r;
  CK(cudaMemcpy(&r, d.es + env, sizeof(EnvS), cudaMemcpyDeviceToHost));
  if (g && (st = gather_vec(sim, d.g, env, g))) return st;
  if (D) {  // elastic + inertia blocks, plus the surface vertices' contact blocks
    std::vector<float> tmp(6 * (size_t)d.nv), tc(6 * (size_t)std::max(1, d.nsv));
    for (int c6 = 0; c6 < 6; ++c6)
      if ((st = copy_env_comp(sim, tmp.data() + (size_t)c6 * d.nv, d.D, env, c6, 6, true))) return st;
    {
      size_t pitch = sizeof(float) * (size_t)(d.Es / 32) * 6 * 32;
      for (int c6 = 0; c6 < 6 && d.nsv > 0; ++c6) {
        size_t off = ((size_t)(env / 32) * 6 + c6) * 32 + (env % 32);
        CK(cudaMemcpy2D(tc.data() + (size_t)c6 * d.nsv, sizeof(float), d.Dcon + off, pitch, sizeof(float), d.nsv,
                        cudaMemcpyDeviceToHost));
      }
    }
    std::vector<int> sl(d.nv, -1);
    for (size_t i = 0; i < sim->sv.size(); ++i) sl[sim->sv[i]] = (int)i;
    for (int v = 0; v < d.nv; ++v) {
      double q[6];
      for (int c6 = 0; c6 < 6; ++c6)
        q[c6] = (double)tmp[(size_t)c6 * d.nv + v] + (sl[v] >= 0 ? (double)tc[(size_t)c6 * d.nsv + sl[v]] : 0.0);
      double M[9] = {q[0], q[3], q[4], q[3], q[1], q[5], q[4], q[5], q[2]};
      for (int k = 0; k < 9; ++k) D[9 * v + k] = M[k];
    }
  }
  if (grig) for (int k = 0; k < 6; ++k) grig[k] = r.gr[k];
  if (Drig) for (int k = 0; k < 9; ++k) { Drig[k] = r.Dc[k]; Drig[9 + k] = r.Dth[k]; }
  if (parts) for (int k = 0; k < 5; ++k) parts[k] = r.Ep[k];
  return post_launch(sim);
}

tac_status tac_debug_iteration(tac_sim* sim, int32_t env, const double* u_t, const double* v_t, const double* c_t,
                               const double* R_t, const double* u, const double* c, const double* R,
                               const double* target7, double dt, const double* g_prev, const double* p_prev,
                               double gPg_prev, int32_t restart, double* p_out, double* out) {
  tac_status st = check_sim(sim);
  if (st) return st;
  if (env < 0 || env >= sim->d.E || !(dt > 0) || !g_prev || !p_prev || !p_out || !out) return TAC_EINVAL;
  // evaluation at x_k (a4, a5, Armijo's first evaluation: accepted)
  if ((st = tac_debug_eval(sim, env, u_t, v_t, c_t, R_t, u, c, R, target7, dt, nullptr, nullptr, nullptr, nullptr,
                           nullptr)))
    return st;
  const Dev& d = sim->d;
  const int nv = d.nv;
  // the previous iterate's gradient and direction (fp32 vectors, fp64 rigid parts)
  if ((st = scatter_vec(sim, d.gp, env, g_prev)) || (st = scatter_vec(sim, d.p, env, p_prev))) return st;
  EnvS es;
  CK(cudaMemcpy(&es, d.es + env, sizeof(EnvS), cudaMemcpyDeviceToHost));
  for (int k = 0; k < 6; ++k) { es.grp[k] = g_prev[3 * nv + k]; es.pr[k] = p_prev[3 * nv + k]; }
  es.gPg_prev = gPg_prev;
  es.restart = restart ? 1 : 0;
  es.iter = 2;  // not the step's first iteration
  es.best_it = 2;
  es.best_pg = INFINITY;
  CK(cudaMemcpy(d.es + env, &es, sizeof(EnvS), cudaMemcpyHostToDevice));
  launch_direction(d, 0);         // a6
  launch_curvature(d, dt, 0);     // a7
  launch_alpha(d, dt, 0);         // a7 / a8
  CK(cudaDeviceSynchronize());
  if ((st = post_launch(sim))) return st;
  CK(cudaMemcpy(&es, d.es + env, sizeof(EnvS), cudaMemcpyDeviceToHost));
  if ((st = gather_vec(sim, d.p, env, p_out))) return st;
  for (int k = 0; k < 6; ++k) p_out[3 * nv + k] = es.pr[k];
  const double r[12] = {es.beta, es.gp_prev, es.gPg_prev, es.beta == 0 ? 1.0 : 0.0, es.dbg[1], es.dbg[3], es.dbg[0],
                        es.dbg[4], es.dbg[5], es.dbg[6], es.dbg[2], es.pg};
  for (int k = 0; k < 12; ++k) out[k] = r[k];
  return TAC_OK;
}

}  // extern "C"
