// kernels.cu — sm_100a kernels of the batched PNCG-IPC step.
//
// Citations: P:L = PAPER.md line L (Supp. §A: P:419-466), R# = DESIGN.md reading.
// Thread mapping:
//   vertex / element kernels: block (32, 8); lane = env (env-fastest SoA), warp = one
//     vertex or tet, so static mesh data is a warp-uniform broadcast load and per-env
//     vertex rows are 128-byte coalesced;
//   contact kernels: blockIdx.y = env, threads stride over that env's candidate pairs;
//   scalar kernels: one thread per env (fp64 control flow of the NCG).
#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "internal.h"

// programmatic dependent launch: wait for the stream predecessor (first statement of
// every kernel; see pdl_launch)
#define TAC_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

namespace tac {

thread_local long long g_launches = 0;
thread_local Profiler* g_prof = nullptr;

static const char* kNames[KID_COUNT] = {
    "step_setup", "vert_setup", "broadphase", "anchors", "vert_pre", "elem_grad", "contact_near_gi", "accept",
    "dir_reduce", "dir_scalar", "dir_apply", "elem_curv", "contact_curv", "alpha", "ccd", "finalize_vert",
    "finalize_env", "markers", "other", "contact_classify", "contact_near_ig", "contact_near_ee",
    "contact_friction", "broadphase_rebuild", "dir_reduce_surf"};
const char* kernel_name(int kid) { return (kid >= 0 && kid < KID_COUNT) ? kNames[kid] : "?"; }

// ------------------------------------------------------------------ small helpers
// AoSoA layout [v][env_group][c][32] (lane = env % 32): the components of one vertex for one
// warp are 128 B apart at compile-time offsets from a single per-vertex base.  32-bit offsets:
// tac_create guarantees 6 nv Es < 2^32.
__device__ __forceinline__ unsigned vidx(const Dev& d, int c, int v, int e) {  // 3-component arrays
  return (((unsigned)v * (unsigned)(d.Es >> 5) + ((unsigned)e >> 5)) * 3u + (unsigned)c) * 32u + ((unsigned)e & 31u);
}
__device__ __forceinline__ unsigned vidxD(const Dev& d, int c, int v, int e) {  // D: 6 components
  return (((unsigned)v * (unsigned)(d.Es >> 5) + ((unsigned)e >> 5)) * 6u + (unsigned)c) * 32u + ((unsigned)e & 31u);
}
__device__ __forceinline__ unsigned vidxS(const Dev& d, int c, int sl, int e) {  // Dcon: 6 per surface vertex
  return (((unsigned)sl * (unsigned)(d.Es >> 5) + ((unsigned)e >> 5)) * 6u + (unsigned)c) * 32u + ((unsigned)e & 31u);
}
// candidate list of env e in buffer b (R16 double buffering)
__device__ __forceinline__ size_t cand_off(const Dev& d, int b, int e) { return ((size_t)b * d.E + e) * d.kmax; }
struct d3 {
  double x, y, z;
};
__device__ __forceinline__ d3 mk(double x, double y, double z) { return d3{x, y, z}; }
__device__ __forceinline__ d3 operator+(d3 a, d3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ d3 operator-(d3 a, d3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ d3 operator*(double s, d3 a) { return mk(s * a.x, s * a.y, s * a.z); }
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ d3 cross(d3 a, d3 b) {
  return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double nrm(d3 a) { return sqrt(dot(a, a)); }
__device__ __forceinline__ d3 mv(const double* R, d3 y) {
  return mk(R[0] * y.x + R[1] * y.y + R[2] * y.z, R[3] * y.x + R[4] * y.y + R[5] * y.z,
            R[6] * y.x + R[7] * y.y + R[8] * y.z);
}
__device__ __forceinline__ d3 ld3(const double* a) { return mk(a[0], a[1], a[2]); }

__device__ __forceinline__ void atomic_max_pos(unsigned* a, float v) {  // v >= 0
  if (v > 0.f) atomicMax(a, __float_as_uint(v));
}
__device__ __forceinline__ void atomic_min_pos(unsigned* a, float v) {
  if (v >= 0.f) atomicMin(a, __float_as_uint(v));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// block-wide sum of one double into *out (atomic), block of up to 1024 threads (1D)
__device__ void block_sum_atomic(double v, double* out, double* sm) {
  v = warp_sum(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    int nw = (blockDim.x + 31) >> 5;
    double s = lane < nw ? sm[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0 && s != 0.0) atomicAdd(out, s);
  }
}

// block-wide sums of N doubles with one __syncthreads: warp shuffles, one row per warp in
// shared memory, then thread k < N sums column k and issues one atomic
template <int N>
__device__ void block_sums_atomic(const double* v, double* const* out, double* sm /* [32][N] */) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double x = warp_sum(v[k]);
    if (lane == 0) sm[w * N + k] = x;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    double s = 0;
    for (int j = 0; j < nw; ++j) s += sm[j * N + threadIdx.x];
    if (s != 0.0) atomicAdd(out[threadIdx.x], s);
  }
}

// the 20 per-env contact accumulators are contiguous: acc[A_EB .. A_DR + 11]
static_assert(A_EF == A_EB + 1 && A_GR == A_EB + 2 && A_DR == A_EB + 8, "accumulator layout");
// warp sums of 20 values by recursive halving: at offset o each lane keeps the half of its
// values selected by (lane & o) and adds the partner's copy of that half, so after offsets
// 16..1 lane L holds the warp total of value L -- 31 double shuffles instead of 20 x 5
__device__ __forceinline__ double warp_sum20_transposed(const double* v) {
  const int lane = threadIdx.x & 31;
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double lo = v[i], hi = i + 16 < 20 ? v[i + 16] : 0.0;
    const bool up = lane & 16;
    a[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, 16);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const bool up = lane & o;
      a[i] = (up ? a[i + o] : a[i]) + __shfl_xor_sync(0xffffffffu, up ? a[i] : a[i + o], o);
    }
  }
  return a[0];
}
__device__ void block_sums_contact(const double* v, double* acc, int Es, int e, double* sm /* [nwarps][20] */) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const double x = warp_sum20_transposed(v);
  if (lane < 20) sm[w * 20 + lane] = x;
  __syncthreads();
  if (threadIdx.x < 20) {
    double s = 0;
    for (int j = 0; j < nw; ++j) s += sm[j * 20 + threadIdx.x];
    if (s != 0.0) atomicAdd(acc + (size_t)(A_EB + threadIdx.x) * Es + e, s);
  }
}

// ---- SO(3), fp64 (R18) ----
__device__ void quat_R(const float* q7, double* R) {
  double w = q7[3], x = q7[4], y = q7[5], z = q7[6];
  double n = sqrt(w * w + x * x + y * y + z * z);
  w /= n; x /= n; y /= n; z /= n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}
__device__ void mm3(const double* A, const double* B, double* C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}
__device__ void mmT(const double* A, const double* B, double* C) {  // A B^T
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[3 * j] + A[3 * i + 1] * B[3 * j + 1] + A[3 * i + 2] * B[3 * j + 2];
}
__device__ void rodrigues(d3 w, double* R) {
  double th = nrm(w);
  double a, b;
  if (th < 1e-8) { a = 1 - th * th / 6; b = 0.5 - th * th / 24; }
  else { a = sin(th) / th; b = (1 - cos(th)) / (th * th); }
  double K[9] = {0, -w.z, w.y, w.z, 0, -w.x, -w.y, w.x, 0};
  double K2[9];
  mm3(K, K, K2);
  for (int i = 0; i < 9; ++i) R[i] = (i % 4 == 0 ? 1.0 : 0.0) + a * K[i] + b * K2[i];
}
__device__ d3 so3_log(const double* R) {
  double tr = R[0] + R[4] + R[8];
  double c = fmax(-1.0, fmin(1.0, 0.5 * (tr - 1)));
  double th = acos(c);
  d3 v = mk(R[7] - R[5], R[2] - R[6], R[3] - R[1]);
  if (th < 1e-6) return (0.5 * (1 + th * th / 6)) * v;
  if (M_PI - th < 1e-6) {
    int i = (R[0] >= R[4] && R[0] >= R[8]) ? 0 : (R[4] >= R[8] ? 1 : 2);
    double a[3];
    a[i] = sqrt(fmax(0.0, 0.5 * (R[4 * i] + 1)));
    for (int j = 0; j < 3; ++j)
      if (j != i) a[j] = (R[3 * i + j] + R[3 * j + i]) / (4 * a[i]);
    d3 ax = mk(a[0], a[1], a[2]);
    return (th / nrm(ax)) * ax;
  }
  return (th / (2 * sin(th))) * v;
}
// force-capped pose spring weight psi'(r)/r (R18)
// J_l(phi)^-T x, J_l the SO(3) left Jacobian: J_l^-1 = I - [phi]/2 + c(t) [phi]^2,
// c(t) = (1 - (t/2) cot(t/2)) / t^2 (-> 1/12); the gradient of lam . log(R R*^T) under
// R <- exp([delta]) R (R29)
__device__ d3 so3_jl_inv_T(d3 phi, d3 x) {
  const double t = nrm(phi);
  const double c = t < 1e-4 ? 1.0 / 12.0 + t * t / 720.0 : (1.0 - 0.5 * t / tan(0.5 * t)) / (t * t);
  const d3 px = cross(phi, x);
  return x + 0.5 * px + c * cross(phi, px);
}
__device__ __forceinline__ double spring_w(double r, double k, double cap) { return r <= cap / k ? k : cap / r; }
__device__ __forceinline__ double spring_e(double r, double k, double cap) {
  double rho = cap / k;
  return r <= rho ? 0.5 * k * r * r : cap * (r - 0.5 * rho);
}

// ---- barrier (R3) and mollifier ----
__device__ __forceinline__ double bar_b(double x, double dh) { return -(x - dh) * (x - dh) * log(x / dh); }
__device__ __forceinline__ double bar_db(double x, double dh) {
  return -2 * (x - dh) * log(x / dh) - (x - dh) * (x - dh) / x;
}
__device__ __forceinline__ double bar_ddb(double x, double dh) {
  return -2 * log(x / dh) - 4 * (x - dh) / x + (x - dh) * (x - dh) / (x * x);
}
__device__ __forceinline__ double moll_f(double s, double eps) {
  return s >= eps ? s : (-s * s * s / (3 * eps * eps) + s * s / eps + eps / 3);
}
__device__ __forceinline__ double moll_f1(double s, double eps) { return s >= eps ? 1.0 / s : (2 / eps - s / (eps * eps)); }

// ---- exact primitive distances, fp64; r = sum_k w_k z_k, d = |r| ----
struct DR {
  double d, w[4];
};
// closest point of segment a + u e (u in [0, 1], inv_ee = 1 / e.e) to p: u and |r|^2
__device__ __forceinline__ double seg_u(d3 p, d3 a, d3 e, double inv_ee) {
  return fmin(1.0, fmax(0.0, dot(p - a, e) * inv_ee));
}
// Same case logic as the oracle (interior solve, else the best boundary candidate), with
// shared reciprocals and squared-distance comparisons: one sqrt per call
__device__ DR dist_pt(d3 p, d3 t0, d3 t1, d3 t2) {
  DR r;
  d3 e1 = t1 - t0, e2 = t2 - t0, q = p - t0;
  double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2), r1 = dot(q, e1), r2 = dot(q, e2);
  double idet = 1.0 / (a11 * a22 - a12 * a12);
  double s = (a22 * r1 - a12 * r2) * idet, t = (a11 * r2 - a12 * r1) * idet;
  if (s >= 0 && t >= 0 && s + t <= 1) {
    r.d = nrm(q - s * e1 - t * e2);
    r.w[0] = 1; r.w[1] = -(1 - s - t); r.w[2] = -s; r.w[3] = -t;
    return r;
  }
  double best = DBL_MAX;
  d3 T[3] = {t0, t1, t2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    int i = k, j = (k + 1) % 3;
    d3 e = T[j] - T[i];
    double u = seg_u(p, T[i], e, 1.0 / dot(e, e));
    d3 v = p - (T[i] + u * e);
    double dd = dot(v, v);
    if (dd < best) {
      best = dd;
      r.w[0] = 1; r.w[1] = 0; r.w[2] = 0; r.w[3] = 0;
      r.w[1 + i] = -(1 - u);
      r.w[1 + j] = -u;
    }
  }
  r.d = sqrt(best);
  return r;
}
__device__ DR dist_ee(d3 a0, d3 a1, d3 b0, d3 b1) {
  DR r;
  d3 d1 = a1 - a0, d2 = b1 - b0, q = a0 - b0;
  double a = dot(d1, d1), e = dot(d2, d2), b = dot(d1, d2), c = dot(d1, q), f = dot(d2, q);
  double den = a * e - b * b;
  if (den > 1e-12 * a * e) {
    double iden = 1.0 / den;
    double s = (b * f - c * e) * iden, t = (a * f - b * c) * iden;
    if (s > 0 && s < 1 && t > 0 && t < 1) {
      r.d = nrm(q + s * d1 - t * d2);
      r.w[0] = 1 - s; r.w[1] = s; r.w[2] = -(1 - t); r.w[3] = -t;
      return r;
    }
  }
  const double ia = 1.0 / a, ie = 1.0 / e;
  double best;
  {
    double t = seg_u(a0, b0, d2, ie);
    d3 v = a0 - (b0 + t * d2);
    best = dot(v, v); r.w[0] = 1; r.w[1] = 0; r.w[2] = -(1 - t); r.w[3] = -t;
  }
  {
    double t = seg_u(a1, b0, d2, ie);
    d3 v = a1 - (b0 + t * d2);
    double dd = dot(v, v);
    if (dd < best) { best = dd; r.w[0] = 0; r.w[1] = 1; r.w[2] = -(1 - t); r.w[3] = -t; }
  }
  {
    double s = seg_u(b0, a0, d1, ia);
    d3 v = (a0 + s * d1) - b0;
    double dd = dot(v, v);
    if (dd < best) { best = dd; r.w[0] = 1 - s; r.w[1] = s; r.w[2] = -1; r.w[3] = 0; }
  }
  {
    double s = seg_u(b1, a0, d1, ia);
    d3 v = (a0 + s * d1) - b1;
    double dd = dot(v, v);
    if (dd < best) { best = dd; r.w[0] = 1 - s; r.w[1] = s; r.w[2] = 0; r.w[3] = -1; }
  }
  r.d = sqrt(best);
  return r;
}

// ---- R33: IPC-toolkit constraint deduplication.  A pair's constraint is its closest features:
// the corners with a non-zero closest-point weight (gel ids surface-local, indenter ids vertex
// ids).  Point-edge and point-point constraints (one side a single vertex, neither side a face,
// not edge-edge) are realised by several pairs; the first pair to claim the constraint's key in
// the env's table carries it (all realisations have the same distance and closest points).
// Returns true for a duplicate.  *interior_ee: an edge-edge constraint (the mollifier's case).
__device__ bool dedup_duplicate(const Dev& d, int e, const unsigned* id, const bool* ind, const double* w,
                                bool* interior_ee) {
  unsigned g[4], y[4];
  int ng = 0, ny = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (w[k] != 0.0) {
      if (ind[k]) y[ny++] = id[k];
      else g[ng++] = id[k];
    }
  const bool shared = ng <= 2 && ny <= 2 && !(ng == 2 && ny == 2);
  *interior_ee = ng == 2 && ny == 2;
  if (!shared) return false;
  const unsigned g0 = ng > 1 ? min(g[0], g[1]) : (ng ? g[0] : 0xffffu), g1 = ng > 1 ? max(g[0], g[1]) : 0xffffu;
  const unsigned y0 = ny > 1 ? min(y[0], y[1]) : (ny ? y[0] : 0xffffu), y1 = ny > 1 ? max(y[0], y[1]) : 0xffffu;
  const unsigned long long key = (unsigned long long)g0 | ((unsigned long long)g1 << 16) |
                                 ((unsigned long long)y0 << 32) | ((unsigned long long)y1 << 48);  // never 0
  unsigned slot = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 52) & (kDedupSlots - 1);
  for (int probe = 0; probe < kDedupSlots; ++probe) {
    unsigned long long* t = d.dtab + (size_t)slot * d.Es + e;
    const unsigned long long prev = atomicCAS(t, 0ull, key);
    if (prev == 0ull) return false;   // claimed: this pair carries the constraint
    if (prev == key) return true;     // another pair carries it
    slot = (slot + 1) & (kDedupSlots - 1);
  }
  d.es[e].ncand_over = 1;  // table full: the step fails (R32)
  return true;
}

// ---- fp32 squared distances on coordinates relative to the pair's first corner: only a
// far/near screen (the same case logic as dist_pt / dist_ee, no weights).  Rounding of the
// relative coordinates and of the case solves stays below ~1e-9 m at pad scale, so a pair
// screened with sqrt(d2) >= dhat + kNearScreen (1e-6 m) is far for the exact distance too.
struct f3 {
  float x, y, z;
};
__device__ __forceinline__ f3 f3sub(f3 a, f3 b) { return f3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ float f3dot(f3 a, f3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ f3 f3axpy(float s, f3 a, f3 b) { return f3{fmaf(s, a.x, b.x), fmaf(s, a.y, b.y), fmaf(s, a.z, b.z)}; }
__device__ __forceinline__ float seg_d2f(f3 p, f3 a, f3 e, float iee) {  // |p - closest point of segment a + u e|^2
  const float u = fminf(1.f, fmaxf(0.f, f3dot(f3sub(p, a), e) * iee));
  const f3 v = f3sub(p, f3axpy(u, e, a));
  return f3dot(v, v);
}
__device__ float dist2_pt_f(f3 p, f3 t0, f3 t1, f3 t2) {
  const f3 e1 = f3sub(t1, t0), e2 = f3sub(t2, t0), q = f3sub(p, t0);
  const float a11 = f3dot(e1, e1), a12 = f3dot(e1, e2), a22 = f3dot(e2, e2), r1 = f3dot(q, e1), r2 = f3dot(q, e2);
  const float idet = 1.f / (a11 * a22 - a12 * a12);
  const float s = (a22 * r1 - a12 * r2) * idet, t = (a11 * r2 - a12 * r1) * idet;
  if (s >= 0.f && t >= 0.f && s + t <= 1.f) {
    const f3 v = f3axpy(-t, e2, f3axpy(-s, e1, q));
    return f3dot(v, v);
  }
  const f3 e3 = f3sub(t2, t1);
  return fminf(fminf(seg_d2f(p, t0, e1, 1.f / a11), seg_d2f(p, t0, e2, 1.f / a22)), seg_d2f(p, t1, e3, 1.f / f3dot(e3, e3)));
}
__device__ float dist2_ee_f(f3 a0, f3 a1, f3 b0, f3 b1) {
  const f3 d1 = f3sub(a1, a0), d2 = f3sub(b1, b0), q = f3sub(a0, b0);
  const float a = f3dot(d1, d1), e = f3dot(d2, d2), b = f3dot(d1, d2), c = f3dot(d1, q), f = f3dot(d2, q);
  const float den = a * e - b * b;
  if (den > 1e-6f * a * e) {
    const float iden = 1.f / den;
    const float s = (b * f - c * e) * iden, t = (a * f - b * c) * iden;
    if (s > 0.f && s < 1.f && t > 0.f && t < 1.f) {
      const f3 v = f3axpy(-t, d2, f3axpy(s, d1, q));
      return f3dot(v, v);
    }
  }
  const float ia = 1.f / a, ie = 1.f / e;
  return fminf(fminf(seg_d2f(a0, b0, d2, ie), seg_d2f(a1, b0, d2, ie)), fminf(seg_d2f(b0, a0, d1, ia), seg_d2f(b1, a0, d1, ia)));
}
// edge-edge mollifier (R30): c = |e_a x e_b|^2 over the corners (a0, a1, b0, b1), eps = 1e-3 La2 Lb2
// (rest squared lengths); m = -c^2/eps^2 + 2c/eps below eps, else 1; dc[k] = dc/dz_k
struct MollD {
  double m, dm;
  d3 dc[4];
};
__device__ MollD ee_moll(const d3* z, double La2, double Lb2) {
  MollD M;
  const d3 ea = z[1] - z[0], eb = z[3] - z[2], w = cross(ea, eb);
  const double c = dot(w, w), eps = 1e-3 * La2 * Lb2;
  const d3 ga = 2.0 * cross(eb, w), gb = 2.0 * cross(w, ea);
  M.dc[0] = -1.0 * ga; M.dc[1] = ga; M.dc[2] = -1.0 * gb; M.dc[3] = gb;
  M.m = 1.0;
  M.dm = 0.0;
  if (c < eps) {
    M.m = (2.0 - c / eps) * c / eps;
    M.dm = (2.0 - 2.0 * c / eps) / eps;
  }
  return M;
}
__device__ __forceinline__ double sqlen4(float4 a, float4 b) {
  const double x = (double)a.x - (double)b.x, y = (double)a.y - (double)b.y, z = (double)a.z - (double)b.z;
  return x * x + y * y + z * z;
}
// corners of a candidate / anchor: ids and sides (gel or indenter)
struct Corners {
  int id[4];
  bool ind[4];
  int na;  // corners on the first side
};
__device__ __forceinline__ Corners corners_of(const Dev& d, int kind, int a, int b) {
  Corners c;
  if (kind == 0) {
    c.id[0] = d.sv[a]; c.ind[0] = false;
    int4 t = d.it[b];
    c.id[1] = t.x; c.id[2] = t.y; c.id[3] = t.z;
    c.ind[1] = c.ind[2] = c.ind[3] = true;
    c.na = 1;
  } else if (kind == 1) {
    c.id[0] = a; c.ind[0] = true;
    int4 t = d.st[b];
    c.id[1] = t.x; c.id[2] = t.y; c.id[3] = t.z;
    c.ind[1] = c.ind[2] = c.ind[3] = false;
    c.na = 1;
  } else {
    int2 ge = d.se[a], ie = d.ie[b];
    c.id[0] = ge.x; c.id[1] = ge.y; c.id[2] = ie.x; c.id[3] = ie.y;
    c.ind[0] = c.ind[1] = false;
    c.ind[2] = c.ind[3] = true;
    c.na = 2;
  }
  return c;
}
struct CornersL {
  int gid[4];  // gel: global vertex id; indenter: vertex id
  int sid[4];  // gel: surface-local index
  bool ind[4];
  int na;
};
__device__ __forceinline__ CornersL corners_l(const Dev& d, int kind, int a, int b) {
  CornersL c;
  if (kind == 0) {
    c.gid[0] = d.sv[a]; c.sid[0] = a; c.ind[0] = false;
    int4 t = d.it[b];
    c.gid[1] = t.x; c.gid[2] = t.y; c.gid[3] = t.z;
    c.ind[1] = c.ind[2] = c.ind[3] = true;
    c.na = 1;
  } else if (kind == 1) {
    c.gid[0] = a; c.ind[0] = true;
    int4 t = d.st[b], tl = d.st_l[b];
    c.gid[1] = t.x; c.gid[2] = t.y; c.gid[3] = t.z;
    c.sid[1] = tl.x; c.sid[2] = tl.y; c.sid[3] = tl.z;
    c.ind[1] = c.ind[2] = c.ind[3] = false;
    c.na = 1;
  } else {
    int2 ge = d.se[a], gl = d.se_l[a], ie = d.ie[b];
    c.gid[0] = ge.x; c.gid[1] = ge.y; c.sid[0] = gl.x; c.sid[1] = gl.y;
    c.gid[2] = ie.x; c.gid[3] = ie.y;
    c.ind[0] = c.ind[1] = false;
    c.ind[2] = c.ind[3] = true;
    c.na = 2;
  }
  return c;
}
// corner ids of a candidate record packed 4 x 16 bit: gel corners by surface-local id,
// indenter corners by vertex id (kind decides which), 16 bits each, the pair's kind in the top
// two bits of the last (nsv, niv < 16384, checked at create): the classification needs no other word
__device__ __forceinline__ uint2 pack_corners(const Dev& d, unsigned long long rec) {
  int kind = (int)(rec >> 62), a = (int)((rec >> 31) & 0x7fffffffu), b = (int)(rec & 0x7fffffffu);
  CornersL C = corners_l(d, kind, a, b);
  unsigned id[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) id[k] = (unsigned)(C.ind[k] ? C.gid[k] : C.sid[k]);
  return make_uint2(id[0] | (id[1] << 16), id[2] | (id[3] << 16) | ((unsigned)kind << 30));
}
__device__ __forceinline__ d3 gel_pos(const Dev& d, const float* u, int v, int e) {
  float4 X = d.X[v];
  return mk((double)X.x + (double)u[vidx(d, 0, v, e)], (double)X.y + (double)u[vidx(d, 1, v, e)],
            (double)X.z + (double)u[vidx(d, 2, v, e)]);
}
__device__ __forceinline__ d3 gel_vec(const Dev& d, const float* a, int v, int e) {
  return mk(a[vidx(d, 0, v, e)], a[vidx(d, 1, v, e)], a[vidx(d, 2, v, e)]);
}
__device__ __forceinline__ d3 ind_body(const Dev& d, int j) {
  float4 y = __ldg(d.Y + j);
  return mk(y.x, y.y, y.z);
}
__device__ __forceinline__ DR pair_dist(int kind, const d3* z) {
  return kind == 2 ? dist_ee(z[0], z[1], z[2], z[3]) : dist_pt(z[0], z[1], z[2], z[3]);
}

// far-pair certificate (R15): world boxes separated along an axis by g >= dhat ->
// separating plane (g, +-e_axis); no barrier term, no exact distance needed
__device__ __forceinline__ bool axis_sep(const d3* z, int na, double dhat, double* g, d3* n) {
  double best = -INFINITY;
  d3 bn = mk(0, 0, 0);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double loA = INFINITY, hiA = -INFINITY, loB = INFINITY, hiB = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double v = a == 0 ? z[k].x : (a == 1 ? z[k].y : z[k].z);
      if (k < na) { loA = fmin(loA, v); hiA = fmax(hiA, v); }
      else { loB = fmin(loB, v); hiB = fmax(hiB, v); }
    }
    if (loA - hiB > best) { best = loA - hiB; bn = mk(a == 0, a == 1, a == 2); }
    if (loB - hiA > best) { best = loB - hiA; bn = mk(-(a == 0), -(a == 1), -(a == 2)); }
  }
  *g = best;
  *n = bn;
  return best >= dhat;
}
// primitive-plane gap (R15, same formula as the oracle's certificate): the supporting
// plane of the triangle (point-triangle) or of both edge directions (edge-edge, unless
// within 1e-3 rad of parallel) holds one side; the other lies |m.(z_A - z_B)|/|m| from it
__device__ __forceinline__ double plane_gap(const d3* z, int na) {
  d3 e1 = z[1] - z[0], e2 = z[3] - z[2], o = z[0] - z[2];
  if (na == 1) { e1 = z[2] - z[1]; e2 = z[3] - z[1]; o = z[0] - z[1]; }
  d3 m = cross(e1, e2);
  double l = nrm(m);
  if (!(l >= 1e-3 * nrm(e1) * nrm(e2) && l > 0)) return -INFINITY;
  return fabs(dot(m, o)) / l;
}
// full far-pair certificate: axis gap, else primitive-plane gap; g = best separation
__device__ __forceinline__ bool far_cert(const d3* z, int na, double dhat, double* g) {
  d3 n;
  if (axis_sep(z, na, dhat, g, &n)) return true;
  *g = fmax(*g, plane_gap(z, na));
  return *g >= dhat;
}

// ------------------------------------------------------------------ a1: step setup
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so env e's noise at step k is a
// pure function of (seed, e, k) -- the same stream in the oracle's own implementation
__device__ void philox4x32_10(uint4 c, uint2 k, unsigned* out) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
    const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  out[0] = c.x; out[1] = c.y; out[2] = c.z; out[3] = c.w;
}
__device__ __forceinline__ double unit_sym(unsigned x) { return ((double)(x >> 8) + 0.5) * (2.0 / 16777216.0) - 1.0; }

// a1: step setup.  R27: with pose noise on, the target of env e at step k is perturbed
// c_s += s_t (u0, u1, u2), R_s <- exp([s_r (u3, u4, u5)]) R_s, u = Philox(seed; e, k, 0 / 1)
__global__ void k_step_setup(Dev d, const float* poses, unsigned long long step) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  EnvS& s = d.es[e];
  const float* q = poses + 7 * e;
  s.cs[0] = q[0]; s.cs[1] = q[1]; s.cs[2] = q[2];
  quat_R(q, s.Rs);
  if (d.noise_t != 0.0 || d.noise_r != 0.0) {
    const unsigned long long gid = (unsigned long long)(e + d.env_offset);
    const uint2 key = make_uint2((unsigned)d.noise_seed, (unsigned)(d.noise_seed >> 32));
    unsigned a[4], b[4];
    philox4x32_10(make_uint4((unsigned)gid, (unsigned)step, (unsigned)(step >> 32), 0u), key, a);
    philox4x32_10(make_uint4((unsigned)gid, (unsigned)step, (unsigned)(step >> 32), 1u), key, b);
    s.cs[0] += d.noise_t * unit_sym(a[0]);
    s.cs[1] += d.noise_t * unit_sym(a[1]);
    s.cs[2] += d.noise_t * unit_sym(a[2]);
    double Q[9], Rn[9];
    rodrigues(mk(d.noise_r * unit_sym(a[3]), d.noise_r * unit_sym(b[0]), d.noise_r * unit_sym(b[1])), Q);
    mm3(Q, s.Rs, Rn);
    for (int i = 0; i < 9; ++i) s.Rs[i] = Rn[i];
  }
  for (int i = 0; i < 3; ++i) { s.c[i] = s.ct[i]; s.cp[i] = s.ct[i]; }
  for (int i = 0; i < 9; ++i) { s.R[i] = s.Rt[i]; s.Rp[i] = s.Rt[i]; }
  double RRt[9];
  mmT(s.Rs, s.Rt, RRt);
  d3 dc = ld3(s.cs) - ld3(s.ct);
  s.flags = (nrm(dc) > 2e-3 || nrm(so3_log(RRt)) > 5 * M_PI / 180) ? 16 : 0;
  s.iter = 0; s.halv = 0; s.restart = 1; s.reeval = 0; s.mode = kActive; s.best_it = 0; s.accepted = 0;
  s.rebuild = 0; s.ncand_over = 0; s.ncand_max = 0; s.nanc_last = 0; s.pending = 0; s.S2 = 0;
  s.odo = 0; s.odo_base = 0; s.Lc = 0; s.cache_ok = 0;
  s.alpha = 0; s.back = 0; s.S = 0; s.best_pg = INFINITY; s.pg = 0; s.E = 0; s.Eprev = 0; s.gp_prev = 0; s.beta = 0;
  for (int i = 0; i < 6; ++i) s.pr[i] = 0;
  d.dalpha[e] = 0.f;
  d.beta[e] = 0.f;
  d.run[e] = 1;
  if (e == 0) { d.anum[0] = -1; d.anum[1] = -1; }  // no active lists yet: identity block mappings
  d.ncand[d.lbuf[e] * d.E + e] = 0;
  d.nanc[e] = 0;
  for (int k = 0; k < kNAcc; ++k) d.acc[(size_t)k * d.Es + e] = 0.0;
  for (int k = 0; k < kNAccU; ++k) d.accu[(size_t)k * d.Es + e] = (k == U_ACCD || k == U_GFAR) ? 0x7f800000u : 0u;
}

// x^ = x^t + h v^t on free vertices; u = u^t
__global__ void k_vert_setup(Dev d, float h) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * 32 + threadIdx.x;
  if (e >= d.E) return;
  for (int v = blockIdx.y * 8 + threadIdx.y; v < d.nv; v += gridDim.y * 8) {
    bool fixed = d.vflag[v] & 1;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      unsigned i = vidx(d, c, v, e);
      float ut = d.ut[i];
      d.u[i] = ut;
      d.uh[i] = fixed ? 0.f : ut + h * d.vt[i];
    }
  }
  if (d.dedup)  // R33: the step-start anchors' constraint table starts empty
    for (int sl = blockIdx.y * 8 + threadIdx.y; sl < kDedupSlots; sl += gridDim.y * 8) d.dtab[(size_t)sl * d.Es + e] = 0ull;
}

// ------------------------------------------------------------------ a2: broad phase
// Candidates (R16): (gel vert, ind tri), (ind vert, gel tri), (gel edge, ind edge) whose
// axis-aligned boxes in the indenter BODY frame are within r on every axis (complete:
// distance >= the largest axis gap in any frame).  Gel vertices go to the body frame
// as b = R^T (x - c) with the oracle's rounding, x = X + u exact in fp64,
// b_a = (R_0a dx_0 + R_1a dx_1) + R_2a dx_2, no contraction (__dmul_rn / __dadd_rn);
// indenter boxes come straight from Y.  The static body-frame BVH is traversed with a
// conservatively inflated fp32 query; leaves run the exact fp64 predicate.
__device__ __forceinline__ double to_body_exact(const double* R, const double* c, d3 x, int a) {
  double d0 = __dsub_rn(x.x, c[0]), d1 = __dsub_rn(x.y, c[1]), d2 = __dsub_rn(x.z, c[2]);
  double t0 = __dmul_rn(R[a], d0), t1 = __dmul_rn(R[3 + a], d1), t2 = __dmul_rn(R[6 + a], d2);
  return __dadd_rn(__dadd_rn(t0, t1), t2);
}

// candidates are staged per WARP in shared memory (its own region and counter) and
// flushed with one global reservation per warp: no block barrier, so a warp whose queries
// run near the indenter never holds up the others
constexpr int kBpWarps = 4;             // 128-thread blocks
constexpr int kBpStageW = 768;          // staged candidates per warp
__shared__ unsigned long long g_bp_sbuf[kBpWarps * kBpStageW];
__shared__ int g_bp_wcnt[kBpWarps];

template <int NIND>
__device__ void bp_query(const Dev& d, int kind, int gid, const double* glo, const double* ghi, double r, int root,
                         unsigned long long* out, uint2* cc, int* cnt, int cap, bool* over) {
  const float eps = 1e-7f;
  float qlo[3], qhi[3];
  for (int a = 0; a < 3; ++a) {
    qlo[a] = (float)(glo[a] - r) - eps;
    qhi[a] = (float)(ghi[a] + r) + eps;
  }
  // kBvhW-wide BVH (child boxes in the parent): a popped node is loaded once and all its
  // children are tested from it, so rejected children and leaves cost no node load
  int stack[48];
  int sp = 0;
  stack[sp++] = root;  // virtual root of the tree
  while (sp > 0) {
    const float4* wn = d.bvhw + kBvhF4 * stack[--sp];
    float4 nd[kBvhF4];
#pragma unroll
    for (int k = 0; k < kBvhF4; ++k) nd[k] = __ldg(wn + k);
#pragma unroll
    for (int chd = 0; chd < kBvhW; ++chd) {
      const float4 n0 = nd[3 * (chd >> 1)], n1 = nd[3 * (chd >> 1) + 1], n2 = nd[3 * (chd >> 1) + 2];
      const bool odd = chd & 1;
      const float lx = odd ? n1.z : n0.x, ly = odd ? n1.w : n0.y, lz = odd ? n2.x : n0.z;
      const float hx = odd ? n2.y : n0.w, hy = odd ? n2.z : n1.x, hz = odd ? n2.w : n1.y;
      if (lx > qhi[0] || hx < qlo[0] || ly > qhi[1] || hy < qlo[1] || lz > qhi[2] || hz < qlo[2]) continue;
      const float4 rq = nd[3 * kBvhW / 2 + (chd >> 2)];
      const float rw = (chd & 3) == 0 ? rq.x : ((chd & 3) == 1 ? rq.y : ((chd & 3) == 2 ? rq.z : rq.w));
      const int rf = __float_as_int(rw);
      if (rf >= 0) { stack[sp++] = rf; continue; }
      const int code = -1 - rf, p0 = code >> 3, np = code & 7;
      for (int k = 0; k < np; ++k) {
        const float4 blo = __ldg(d.bvh_pbox + 2 * (p0 + k)), bhi = __ldg(d.bvh_pbox + 2 * (p0 + k) + 1);
        const int prim = __float_as_int(blo.w);
        // exact prim box (min / max of its float Y corners), tested in double as before
        const double lo[3] = {blo.x, blo.y, blo.z}, hi[3] = {bhi.x, bhi.y, bhi.z};
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 3; ++a)
          if (glo[a] > __dadd_rn(hi[a], r) || lo[a] > __dadd_rn(ghi[a], r)) ok = false;
        if (!ok) continue;
        unsigned long long a_id = (kind == 1) ? (unsigned long long)prim : (unsigned long long)gid;
        unsigned long long b_id = (kind == 1) ? (unsigned long long)gid : (unsigned long long)prim;
        const unsigned long long rec = ((unsigned long long)kind << 62) | (a_id << 31) | b_id;
        const int w = threadIdx.x >> 5;
        int ss = atomicAdd(&g_bp_wcnt[w], 1);  // warp-local staging (native shared int atomic)
        if (ss < kBpStageW) {
          g_bp_sbuf[w * kBpStageW + ss] = rec;
        } else {  // staging full: reserve directly
          int slot = atomicAdd(cnt, 1);
          if (slot < cap) {
            out[slot] = rec;
            if (cc) cc[slot] = pack_corners(d, rec);
          } else {
            *over = true;
          }
        }
      }
    }
  }
}

// flush this warp's staged candidates (all 32 lanes call it, convergent)
__device__ void bp_flush_warp(const Dev& d, unsigned long long* out, uint2* cc, int* cnt, int cap, bool* over) {
  __syncwarp();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = min(g_bp_wcnt[w], kBpStageW);
  int base = 0;
  if (lane == 0 && n) base = atomicAdd(cnt, n);
  base = __shfl_sync(0xffffffffu, base, 0);
  const unsigned long long* sb = g_bp_sbuf + w * kBpStageW;
  for (int j = lane; j < n; j += 32) {
    if (base + j < cap) {
      out[base + j] = sb[j];
      if (cc) cc[base + j] = pack_corners(d, sb[j]);
    } else {
      *over = true;
    }
  }
  __syncwarp();
  if (lane == 0) g_bp_wcnt[w] = 0;
  __syncwarp();
}

// candidates of gel-surface primitives [i0, i1) (strided) of env e.  Called by whole
// warps (lane i0 = warp base + lane, uniform stride); between rounds the warp flushes its
// staging region once it is half full
__device__ void bp_range(const Dev& d, int e, int i0, int i1, int stride, double r, unsigned long long* out, uint2* cc,
                         int* cnt, int cap, const double* R, const double* c) {
  bool over = false;
  const int lane = threadIdx.x & 31;
  for (int b = i0 - lane; b < i1; b += stride) {
    const int i = b + lane;
    if (i < i1) {
    int vv[3], nvx, kind, gid, root;
    if (i < d.nsv) {
      vv[0] = d.sv[i]; nvx = 1; kind = 0; gid = i; root = 0;  // virtual wide roots: 0 tri, 1 edge, 2 vert
    } else if (i < d.nsv + d.nse) {
      gid = i - d.nsv;
      int2 ed = d.se[gid];
      vv[0] = ed.x; vv[1] = ed.y; nvx = 2; kind = 2; root = 1;
    } else {
      gid = i - d.nsv - d.nse;
      int4 t = d.st[gid];
      vv[0] = t.x; vv[1] = t.y; vv[2] = t.z; nvx = 3; kind = 1; root = 2;
    }
    double lo[3], hi[3];
    for (int j = 0; j < nvx; ++j) {
      d3 x = gel_pos(d, d.u, vv[j], e);
      for (int a = 0; a < 3; ++a) {
        double b = to_body_exact(R, c, x, a);
        lo[a] = j ? fmin(lo[a], b) : b;
        hi[a] = j ? fmax(hi[a], b) : b;
      }
    }
    if (kind == 0) bp_query<3>(d, 0, gid, lo, hi, r, root, out, cc, cnt, cap, &over);
    else if (kind == 2) bp_query<2>(d, 2, gid, lo, hi, r, root, out, cc, cnt, cap, &over);
    else bp_query<1>(d, 1, gid, lo, hi, r, root, out, cc, cnt, cap, &over);
    }
    __syncwarp();
    if (g_bp_wcnt[threadIdx.x >> 5] > kBpStageW / 2) bp_flush_warp(d, out, cc, cnt, cap, &over);
  }
  if (over) d.es[e].ncand_over = 1;
}



__global__ void __launch_bounds__(128) k_broadphase(Dev d, double r, unsigned long long* out_override,
                                                    int* cnt_override, int cap_override) {
  TAC_PDL_WAIT();
  int e = blockIdx.y;
  if (e >= d.E) return;
  const EnvS& s = d.es[e];
  if (s.mode != kActive) return;
  __shared__ double R[9], c[3];
  if (threadIdx.x < 9) R[threadIdx.x] = s.R[threadIdx.x];
  if (threadIdx.x < 3) c[threadIdx.x] = s.c[threadIdx.x];
  if (threadIdx.x < kBpWarps) g_bp_wcnt[threadIdx.x] = 0;
  __syncthreads();  // the only block barrier: R, c and the counters before any query
  const int lb = d.lbuf[e];
  unsigned long long* out = out_override ? out_override : d.cand + cand_off(d, lb, e);
  int* cnt = cnt_override ? cnt_override : d.ncand + lb * d.E + e;
  int cap = out_override ? cap_override : d.kmax;
  uint2* cc = out_override ? nullptr : d.ccorn + cand_off(d, lb, e);
  int ntot = d.nsv + d.nse + d.nst;
  if (!out_override && blockIdx.x == 0 && threadIdx.x == 0) d.es[e].cache_ok = 0;  // new candidate list
  bp_range(d, e, blockIdx.x * blockDim.x + threadIdx.x, ntot, gridDim.x * blockDim.x, r, out, cc, cnt, cap, R, c);
  bool over = false;
  bp_flush_warp(d, out, cc, cnt, cap, &over);
  if (over) d.es[e].ncand_over = 1;
}

// ---- initial-pose validation (tac_create): does any gel surface edge cross an indenter
// triangle?  Unsigned distances cannot see a deep intersection (crossing surfaces have
// small positive distances), so tac_create also runs this fp64 segment-triangle test on
// the wide triangle BVH in the body frame.  (An indenter spike piercing one gel triangle
// without any gel edge crossing an indenter triangle is not detected.)
__device__ __forceinline__ double orient3(d3 a, d3 b, d3 c, d3 p) { return dot(cross(b - a, c - a), p - a); }
__global__ void __launch_bounds__(128) k_intersect_check(Dev d, int* hit) {
  TAC_PDL_WAIT();
  const int e = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E || i >= d.nse) return;
  const EnvS& s = d.es[e];
  double R[9], c[3];
  for (int k = 0; k < 9; ++k) R[k] = s.R[k];
  for (int k = 0; k < 3; ++k) c[k] = s.c[k];
  const int2 ed = d.se[i];
  const d3 x0 = gel_pos(d, d.u, ed.x, e), x1 = gel_pos(d, d.u, ed.y, e);
  const d3 p0 = mk(to_body_exact(R, c, x0, 0), to_body_exact(R, c, x0, 1), to_body_exact(R, c, x0, 2));
  const d3 p1 = mk(to_body_exact(R, c, x1, 0), to_body_exact(R, c, x1, 1), to_body_exact(R, c, x1, 2));
  const float qlo[3] = {(float)fmin(p0.x, p1.x) - 1e-6f, (float)fmin(p0.y, p1.y) - 1e-6f, (float)fmin(p0.z, p1.z) - 1e-6f};
  const float qhi[3] = {(float)fmax(p0.x, p1.x) + 1e-6f, (float)fmax(p0.y, p1.y) + 1e-6f, (float)fmax(p0.z, p1.z) + 1e-6f};
  int stack[48];
  int sp = 0;
  stack[sp++] = 0;  // virtual root of the triangle BVH
  while (sp > 0) {
    const float4* wn = d.bvhw + kBvhF4 * stack[--sp];
    float4 nd[kBvhF4];
#pragma unroll
    for (int k = 0; k < kBvhF4; ++k) nd[k] = __ldg(wn + k);
#pragma unroll
    for (int chd = 0; chd < kBvhW; ++chd) {
      const float4 n0 = nd[3 * (chd >> 1)], n1 = nd[3 * (chd >> 1) + 1], n2 = nd[3 * (chd >> 1) + 2];
      const bool odd = chd & 1;
      const float lx = odd ? n1.z : n0.x, ly = odd ? n1.w : n0.y, lz = odd ? n2.x : n0.z;
      const float hx = odd ? n2.y : n0.w, hy = odd ? n2.z : n1.x, hz = odd ? n2.w : n1.y;
      if (lx > qhi[0] || hx < qlo[0] || ly > qhi[1] || hy < qlo[1] || lz > qhi[2] || hz < qlo[2]) continue;
      const float4 rq = nd[3 * kBvhW / 2 + (chd >> 2)];
      const float rw = (chd & 3) == 0 ? rq.x : ((chd & 3) == 1 ? rq.y : ((chd & 3) == 2 ? rq.z : rq.w));
      const int rf = __float_as_int(rw);
      if (rf >= 0) { stack[sp++] = rf; continue; }
      const int code = -1 - rf, q0 = code >> 3, nq = code & 7;
      for (int k = 0; k < nq; ++k) {
        const int prim = __float_as_int(__ldg(d.bvh_pbox + 2 * (q0 + k)).w);
        const int4 t = d.it[prim];
        const d3 a = ind_body(d, t.x), b = ind_body(d, t.y), cc = ind_body(d, t.z);
        const double s0 = orient3(a, b, cc, p0), s1 = orient3(a, b, cc, p1);
        if (!((s0 < 0 && s1 > 0) || (s0 > 0 && s1 < 0))) continue;  // both ends on one side
        const double o0 = orient3(p0, p1, a, b), o1 = orient3(p0, p1, b, cc), o2 = orient3(p0, p1, cc, a);
        if ((o0 >= 0 && o1 >= 0 && o2 >= 0) || (o0 <= 0 && o1 <= 0 && o2 <= 0)) {
          atomicExch(hit + e, 1);
          return;
        }
      }
    }
  }
}

// rebuilds inside the loop: only the envs k_alpha listed; work items = (listed env,
// 32-primitive chunk) per WARP over a fixed grid, so cost follows the actual rebuild count
// and no warp waits for another
// rebuild work items carry kRebuildChunk primitives per warp (lanes beyond it idle): the
// launch is set by its slowest warp, a warp executes the union of its lanes' divergent BVH
// paths, and the rebuild has far fewer items than warp slots -- thinner items, shorter tail
__global__ void __launch_bounds__(128) k_broadphase_list(Dev d, double r, int kRebuildChunk) {
  TAC_PDL_WAIT();
  const int nreb = *d.nreb;
  const int ntot = d.nsv + d.nse + d.nst;
  const int nchunk = (ntot + kRebuildChunk - 1) / kRebuildChunk;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double Rw[kBpWarps][12];  // per-warp R, c of its current env
  if (lane == 0) g_bp_wcnt[w] = 0;
  __syncwarp();
  const int nw = gridDim.x * kBpWarps;
  for (int item = blockIdx.x * kBpWarps + w; item < nreb * nchunk; item += nw) {
    const int e = d.reb_list[item / nchunk], ch = item % nchunk;
    const EnvS& s = d.es[e];
    // the pending buffer, at the build point's pose (k_alpha's trial: k_accept may move s.c, s.R
    // while this runs concurrently with the evaluation)
    const int nb = 1 - d.lbuf[e];
    if (lane < 9) Rw[w][lane] = s.Rb[lane];
    else if (lane < 12) Rw[w][lane] = s.cb[lane - 9];
    __syncwarp();
    unsigned long long* cd = d.cand + cand_off(d, nb, e);
    uint2* cc = d.ccorn + cand_off(d, nb, e);
    int* cn = d.ncand + nb * d.E + e;
    bp_range(d, e, ch * kRebuildChunk + lane, min(ntot, (ch + 1) * kRebuildChunk), ntot, r, cd, cc, cn, d.kmax, Rw[w],
             Rw[w] + 9);  // one round: prims [Q ch, Q ch + Q)
    bool over = false;
    bp_flush_warp(d, cd, cc, cn, d.kmax, &over);
    if (over) d.es[e].ncand_over = 1;
  }
}

// ------------------------------------------------------------------ a3: friction anchors
// pairs with d(x^t) < dhat: lambda = -kappa b'(d), frozen weights, tangent basis (R7)
__global__ void k_anchors(Dev d, double h2) {
  TAC_PDL_WAIT();
  int e = blockIdx.y;
  if (e >= d.E || d.es[e].mode != kActive) return;
  const EnvS& s = d.es[e];
  const double kappa = h2 * d.edbl[e];  // h^2 kappa_phys of this env
  const int lb = d.lbuf[e];
  int n = min(d.ncand[lb * d.E + e], d.kmax);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long rec = d.cand[cand_off(d, lb, e) + i];
    int kind = (int)(rec >> 62), a = (int)((rec >> 31) & 0x7fffffffu), b = (int)(rec & 0x7fffffffu);
    Corners C = corners_of(d, kind, a, b);
    d3 z[4];
    for (int k = 0; k < 4; ++k) z[k] = C.ind[k] ? mv(s.R, ind_body(d, C.id[k])) + ld3(s.c) : gel_pos(d, d.u, C.id[k], e);
    DR D = pair_dist(kind, z);
    if (!(D.d < d.dhat) || !(D.d > 0)) continue;
    CornersL L = corners_l(d, kind, a, b);
    bool ee_int = true;
    if (d.dedup) {  // R33: one anchor per constraint (ids: gel surface-local, indenter vertex)
      unsigned kid[4];
      for (int k = 0; k < 4; ++k) kid[k] = C.ind[k] ? (unsigned)C.id[k] : (unsigned)L.sid[k];
      if (dedup_duplicate(d, e, kid, C.ind, D.w, &ee_int)) continue;
    }
    d3 rr = mk(0, 0, 0);
    for (int k = 0; k < 4; ++k) rr = rr + D.w[k] * z[k];
    d3 nn = (1.0 / D.d) * rr;
    double ax = fabs(nn.x), ay = fabs(nn.y), az = fabs(nn.z);
    d3 ee = (ax <= ay && ax <= az) ? mk(1, 0, 0) : (ay <= az ? mk(0, 1, 0) : mk(0, 0, 1));
    d3 t1 = cross(nn, ee);
    t1 = (1.0 / nrm(t1)) * t1;
    d3 t2 = cross(nn, t1);
    int slot = atomicAdd(d.nanc + e, 1);
    if (slot >= d.amax) { d.es[e].ncand_over = 1; continue; }
    Anchor A;
    int ng = 0;
    unsigned sid[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k) { A.gid[k] = -1; A.w[k] = 0.f; }
    A.t1[0] = t1.x; A.t1[1] = t1.y; A.t1[2] = t1.z;
    A.t2[0] = t2.x; A.t2[1] = t2.y; A.t2[2] = t2.z;
    double mol = 1.0;
    if (kind == 2 && d.ee_moll && ee_int)  // R30: lambda of the mollified edge-edge barrier
      mol = ee_moll(z, sqlen4(__ldg(d.X + C.id[1]), __ldg(d.X + C.id[0])),
                    sqlen4(__ldg(d.Y + C.id[3]), __ldg(d.Y + C.id[2]))).m;
    A.lam = (float)fmax(0.0, -mol * kappa * bar_db(D.d, d.dhat));
    A.pad2 = 0; A.pad3 = 0;
    // fold the rigid side: Y_w = sum_ind w Y, sig = sum_ind w; C0 = sum_gel w u^t + R^t Y_w + sig c^t.
    // Fixed gel corners are dropped: u = 0 there, so they add nothing to Delta and take no force
    d3 yw = mk(0, 0, 0), c0 = mk(0, 0, 0);
    double sig = 0;
    for (int k = 0; k < 4; ++k) {
      const float wf = (float)D.w[k];
      const double wk = (double)wf;
      if (C.ind[k]) { yw = yw + wk * ind_body(d, C.id[k]); sig += wk; }
      else if (!(d.vflag[C.id[k]] & 1)) {
        c0 = c0 + wk * gel_vec(d, d.u, C.id[k], e);
        A.gid[ng] = C.id[k]; A.w[ng] = wf; sid[ng] = (unsigned)L.sid[k]; ++ng;
      }
    }
    A.sid01 = sid[0] | (sid[1] << 16);
    A.sid2 = sid[2];
    A.sig = (float)sig;
    A.yw[0] = (float)yw.x; A.yw[1] = (float)yw.y; A.yw[2] = (float)yw.z;
    // C0 from the stored (rounded) Y_w and sig, so Delta(x^t) = 0 exactly
    c0 = c0 + mv(s.R, mk(A.yw[0], A.yw[1], A.yw[2])) + (double)A.sig * ld3(s.c);
    A.c0[0] = c0.x; A.c0[1] = c0.y; A.c0[2] = c0.z;
    d.anc[(size_t)e * d.amax + slot] = A;
  }
}

// ------------------------------------------------------------------ a4: vertex pre-pass
// applies the pending update u += dalpha p (a8), then the inertia term
// 1/2 m |u - u^|^2, g = m (u - u^), D = m I (lumped M)
// ---- env-group grids of the vertex and element passes (one block dimension = the Es / 32
// groups of 32 envs, the other = chunks of the vertex / cell loop).  In the tolerance mode, once
// at most half the groups hold an env of k_alpha's list, the blocks of the idle groups are dealt
// to the listed groups (each gets up to cap chunks instead of its own row of the grid); otherwise
// (and in the fixed mode) the mapping is the identity.  ng_grid: the group index of this block
// in the launch grid, nc / c: chunks per group and this block's chunk.
__device__ __forceinline__ bool group_block(const Dev& d, int cap, int ng_grid, int c, int nc, int& grp, int& bc,
                                            int& nbc) {
  grp = ng_grid;
  bc = c;
  nbc = nc;
  const int G = d.Es >> 5;
  if (d.fixed_iters > 0 || G < 2 || nc >= cap) return true;
  const int n_g = d.anum[1];
  if (n_g <= 0 || 2 * n_g > G) return true;
  const int per = min(cap, (G * nc) / n_g);
  if (per <= nc) return true;
  const int lin = ng_grid * nc + c, idx = lin / per;
  if (idx >= n_g) return false;
  bc = lin - idx * per;
  nbc = per;
  grp = d.glist[idx];
  return true;
}

// Lane -> env of the vertex / element passes.  As group_block, and in addition: in the tolerance
// mode, once the listed envs are sparse in their groups (on average <= d.compact of 32 lanes), the
// passes run over compacted groups -- lane l of compacted group j is env alist[32 j + l] (lanes
// past the list get e = E: inactive) -- so a warp serves 32 envs that still iterate instead of a
// few: the element passes are instruction-bound, and the scattered per-lane rows cost L2
// requests, not bytes.  Otherwise e = 32 grp + lane.
template <bool TOL>  // TOL: the tolerance mode's instantiation (the fixed mode's is the identity)
__device__ __forceinline__ bool env_lanes(const Dev& d, int cap, int ng_grid, int c, int nc, int& e, int& bc,
                                          int& nbc) {
  const int lane = threadIdx.x & 31;
  if constexpr (!TOL) {
    bc = c;
    nbc = nc;
    e = ng_grid * 32 + lane;
    return true;
  }
  const int G = d.Es >> 5;
  if (G >= 2 && d.compact) {
    const int n = d.anum[0], n_g = d.anum[1];
    if (n > 0 && n <= n_g * d.compact) {  // on average <= d.compact listed lanes per listed group
      const int Gc = (n + 31) >> 5;
      const int per = max(nc, min(cap, (G * nc) / Gc));
      const int lin = ng_grid * nc + c, idx = lin / per;
      if (idx >= Gc) return false;
      bc = lin - idx * per;
      nbc = per;
      const int j = 32 * idx + lane;
      e = j < n ? d.alist[j] : d.E;
      return true;
    }
  }
  int grp;
  if (!group_block(d, cap, ng_grid, c, nc, grp, bc, nbc)) return false;
  e = grp * 32 + lane;
  return true;
}

template <bool TOL>
__global__ void k_vert_pre(Dev d, float h2) {
  TAC_PDL_WAIT();
  int e, by, nby;
  if (!env_lanes<TOL>(d, (d.nv + 7) / 8, blockIdx.x, blockIdx.y, gridDim.y, e, by, nby)) return;
  bool act = e < d.E && (d.run[e] & 1);
  if (!__any_sync(0xffffffffu, act)) return;
  float da = act ? d.dalpha[e] : 0.f;
  if (act && by == 0 && threadIdx.y == 0) {  // near lists are rebuilt by the contact classification
    d.nnear[3 * e] = 0; d.nnear[3 * e + 1] = 0; d.nnear[3 * e + 2] = 0;
    EnvS& s = d.es[e];
    if (s.pending && s.iter >= s.reb_iter + 1) {  // R16 pipeline: the list rebuilt during the last
                                                    // evaluation becomes the active one
      d.lbuf[e] ^= 1;
      s.S = s.S2;
      s.pending = 0;
      s.cache_ok = 0;
      s.ncand_max = max(s.ncand_max, d.ncand[d.lbuf[e] * d.E + e]);
    }
  }
  double ein = 0;
  // two vertices per iteration, every load issued before any store (the stores to u
  // could otherwise alias the next loads and serialise them): twice the bytes in flight
  const int stride = nby * 8;
  for (int v0 = by * 8 + threadIdx.y; v0 < d.nv; v0 += 2 * stride) {
    float u[2][3], pv[2][3], uh[2][3], m[2], sm[2];
    int si[2];
    bool ok[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int v = v0 + t * stride;
      ok[t] = act && v < d.nv && !(d.vflag[v] & 1);
      if (!ok[t]) continue;
      m[t] = d.mass[v] * d.emat[2 * d.Es + e];  // per-env density and shear modulus scales
      sm[t] = d.smu[v] * d.emat[3 * d.Es + e];
      si[t] = d.sidx[v];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned i = vidx(d, c, v, e);
        u[t][c] = d.u[i];
        uh[t][c] = d.uh[i];
        pv[t][c] = da != 0.f ? d.p[i] : 0.f;
      }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (!ok[t]) continue;
      const int v = v0 + t * stride;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned i = vidx(d, c, v, e);
        float uu = u[t][c];
        if (da != 0.f) {
          uu = uu + da * pv[t][c];
          d.u[i] = uu;
        }
        const float du = uu - uh[t][c];
        ein += 0.5 * (double)m[t] * (double)du * (double)du;
        d.g[i] = m[t] * du;
        u[t][c] = uu;
      }
      if (si[t] >= 0) {
        d.usurf[(size_t)si[t] * d.Es + e] = make_float4(u[t][0], u[t][1], u[t][2], 0.f);
#pragma unroll
        for (int c = 0; c < 6; ++c) d.Dcon[vidxS(d, c, si[t], e)] = 0.f;
      }
      const float dg = m[t] + h2 * sm[t];  // mass + state-independent elastic diagonal (App. B)
      d.D[vidxD(d, 0, v, e)] = dg;
      d.D[vidxD(d, 1, v, e)] = dg;
      d.D[vidxD(d, 2, v, e)] = dg;
      d.D[vidxD(d, 3, v, e)] = 0.f;
      d.D[vidxD(d, 4, v, e)] = 0.f;
      d.D[vidxD(d, 5, v, e)] = 0.f;
    }
  }
  if (act && ein != 0.0) atomicAdd(d.acc + (size_t)A_EIN * d.Es + e, ein);
  if (d.dedup && act)  // R33: this evaluation's constraint table starts empty
    for (int sl = by * 8 + threadIdx.y; sl < kDedupSlots; sl += nby * 8) d.dtab[(size_t)sl * d.Es + e] = 0ull;
}

// ------------------------------------------------------------------ a4: element gradient
// Stable Neo-Hookean (R1) on displacements: G = sum_k (u_k - u_0) b_k^T, F = I + G,
//   Psi = mu (|G|^2/2 - i2(G) - det G) + lambda'/2 (J-1)^2,  J-1 = trG + i2 + detG
//   P = mu (G + G^T - trG I - cof G) + lambda'(J-1) cof F
//   f_k = h^2 V P b_k,  D_kk += h^2 V (mu |b_k|^2 I + lambda' c_k c_k^T),  c_k = cof(F) b_k
// (cancellation-free forms of Psi, P; App. B diagonal blocks, exact and PSD)
struct TetData {
  float b[3][3];
  float vol;
};
__device__ __forceinline__ TetData load_tet(const Dev& d, int t) {
  TetData T;
  float4 r0 = __ldg(d.tetb + 3 * t), r1 = __ldg(d.tetb + 3 * t + 1), r2 = __ldg(d.tetb + 3 * t + 2);
  T.b[0][0] = r0.x; T.b[0][1] = r0.y; T.b[0][2] = r0.z; T.vol = r0.w;
  T.b[1][0] = r1.x; T.b[1][1] = r1.y; T.b[1][2] = r1.z;
  T.b[2][0] = r2.x; T.b[2][1] = r2.y; T.b[2][2] = r2.z;
  return T;
}
__device__ __forceinline__ void cof33(const float* A, float* C) {
  C[0] = A[4] * A[8] - A[5] * A[7]; C[1] = A[5] * A[6] - A[3] * A[8]; C[2] = A[3] * A[7] - A[4] * A[6];
  C[3] = A[2] * A[7] - A[1] * A[8]; C[4] = A[0] * A[8] - A[2] * A[6]; C[5] = A[1] * A[6] - A[0] * A[7];
  C[6] = A[1] * A[5] - A[2] * A[4]; C[7] = A[2] * A[3] - A[0] * A[5]; C[8] = A[0] * A[4] - A[1] * A[3];
}

__global__ void __launch_bounds__(256, 4) k_elem_grad(Dev d, float h2) {
  TAC_PDL_WAIT();
  // env group = blockIdx.y (slowest) so the g / D lines of the env groups in flight stay in L2
  const int e = blockIdx.y * 32 + threadIdx.x;
  const bool act = e < d.E && (d.run[e] & 1);
  if (!__any_sync(0xffffffffu, act)) return;
  const float mu = d.emat[e], l2 = d.emat[d.Es + e];  // per-env material
  // AoSoA: one per-vertex base, components at immediate offsets of 32 floats
  const unsigned G = (unsigned)(d.Es >> 5), eg = (unsigned)blockIdx.y, lane = threadIdx.x;
  const float* __restrict__ up = d.u;
  float* __restrict__ gp = d.g;
  float* __restrict__ Dp = d.D;
  double esum = 0;
  for (int it = blockIdx.x * 8 + threadIdx.y; it < d.nrest; it += gridDim.x * 8) {
    const int t = __ldg(d.rest_tets + it);  // tets not covered by k_elem_grad_cells
    int4 tv = __ldg(d.tets + t);
    TetData T = load_tet(d, t);
    const unsigned fixmask = __float_as_uint(__ldg(d.tetb + 3 * t + 1).w);  // bit k: corner k fixed
    if (!act) continue;
    const unsigned vb[4] = {(unsigned)tv.x * G + eg, (unsigned)tv.y * G + eg, (unsigned)tv.z * G + eg,
                            (unsigned)tv.w * G + eg};
    float uu[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float* p = up + (vb[k] * 3u * 32u + lane);
#pragma unroll
      for (int c = 0; c < 3; ++c) uu[k][c] = p[32 * c];
    }
    float G[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) s = fmaf(uu[k + 1][i] - uu[0][i], T.b[k][j], s);
        G[3 * i + j] = s;
      }
    float trG = G[0] + G[4] + G[8];
    float i2 = (G[0] * G[4] - G[1] * G[3]) + (G[0] * G[8] - G[2] * G[6]) + (G[4] * G[8] - G[5] * G[7]);
    float cG[9];
    cof33(G, cG);
    float detG = G[0] * cG[0] + G[1] * cG[1] + G[2] * cG[2];
    float Jm1 = trG + i2 + detG;
    float GG = 0.f;
#pragma unroll
    for (int i = 0; i < 9; ++i) GG = fmaf(G[i], G[i], GG);
    float w = h2 * T.vol;
    esum += (double)(w * (mu * (0.5f * GG - i2 - detG) + 0.5f * l2 * Jm1 * Jm1));
    // cof F = (1 + trG) I - G^T + cof G;  P(F) = mu (G + G^T - trG I - cof G) + lambda'(J-1) cof F
    float cF[9], PK[9];
    const float lj = l2 * Jm1;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        cF[3 * i + j] = (i == j ? 1.f + trG : 0.f) - G[3 * j + i] + cG[3 * i + j];
        PK[3 * i + j] = w * (mu * (G[3 * i + j] + G[3 * j + i] - (i == j ? trG : 0.f) - cG[3 * i + j]) + lj * cF[3 * i + j]);
      }
    float f[4][3], cv[4][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { f[0][c] = 0.f; cv[0][c] = 0.f; }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        float fi = PK[3 * i] * T.b[k][0] + PK[3 * i + 1] * T.b[k][1] + PK[3 * i + 2] * T.b[k][2];
        float ci = cF[3 * i] * T.b[k][0] + cF[3 * i + 1] * T.b[k][1] + cF[3 * i + 2] * T.b[k][2];
        f[k + 1][i] = fi;
        cv[k + 1][i] = ci;
        f[0][i] -= fi;
        cv[0][i] -= ci;
      }
    // diagonal blocks: the state-independent mu |b_k|^2 I part is precomputed per vertex (smu,
    // added with the mass in k_vert_pre); here only lambda' c_k c_k^T
    const float lc = w * l2;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (fixmask & (1u << k)) continue;
      float* pg = gp + (vb[k] * 3u * 32u + lane);
      float* pd = Dp + (vb[k] * 6u * 32u + lane);
      atomicAdd(pg, f[k][0]);
      atomicAdd(pg + 32, f[k][1]);
      atomicAdd(pg + 64, f[k][2]);
      const float sx = lc * cv[k][0], sy = lc * cv[k][1];
      atomicAdd(pd, sx * cv[k][0]);
      atomicAdd(pd + 32, sy * cv[k][1]);
      atomicAdd(pd + 64, lc * cv[k][2] * cv[k][2]);
      atomicAdd(pd + 96, sx * cv[k][1]);
      atomicAdd(pd + 128, sx * cv[k][2]);
      atomicAdd(pd + 160, sy * cv[k][2]);
    }
  }
  if (act) atomicAdd(d.acc + (size_t)A_EEL * d.Es + e, esum);
}

// ---- Kuhn-cell element gradient: one warp = one cell (6 tets, 8 corners) x 32 envs ----
// The 8 corners' u and their 8 x 9 accumulators live in registers with compile-time
// indexing (canonical corner pattern kCellTet), so a cell costs 24 row loads and <= 72
// coalesced red.add instead of 72 and 216 for six independent tets.
// canonical tets (corner slots): {0,1,3,7} {0,1,5,7} {0,2,3,7} {0,2,6,7} {0,4,5,7} {0,4,6,7}
#define CELL_TET(j, k) ((k) == 0 ? 0 : (k) == 3 ? 7 : (j) < 2 ? ((k) == 1 ? 1 : ((j) == 0 ? 3 : 5)) \
                        : (j) < 4 ? ((k) == 1 ? 2 : ((j) == 2 ? 3 : 6)) : ((k) == 1 ? 4 : ((j) == 4 ? 5 : 6)))
// corner bit flipped along step i of tet j's path 0 -> CELL_TET(j,1) -> CELL_TET(j,2) -> 7
#define CELL_Q(j, i) ((i) == 0 ? ((j) >> 1) : (i) == 1 ? (((j) >> 1) == 0 ? 1 + ((j) & 1) : ((j) >> 1) == 1 ? 2 * ((j) & 1) : ((j) & 1)) \
                      : 3 - ((j) >> 1) - (((j) >> 1) == 0 ? 1 + ((j) & 1) : ((j) >> 1) == 1 ? 2 * ((j) & 1) : ((j) & 1)))
// ---- packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2): one instruction evaluates the same
// operation for two tets of a Kuhn cell (.x, .y), halving the issue slots of the elementwise
// 3x3 algebra; each lane rounds exactly like the scalar instruction
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fms2(float2 a, float2 b, float2 c) {  // c - a b
  return __ffma2_rn(make_float2(-a.x, -a.y), b, c);
}
__device__ __forceinline__ float2 det2x2_2(float2 a, float2 b, float2 c, float2 e) { return fms2(c, e, mul2(a, b)); }  // ab - ce
__device__ __forceinline__ void cof33_2(const float2* A, float2* C) {
  C[0] = det2x2_2(A[4], A[8], A[5], A[7]); C[1] = det2x2_2(A[5], A[6], A[3], A[8]); C[2] = det2x2_2(A[3], A[7], A[4], A[6]);
  C[3] = det2x2_2(A[2], A[7], A[1], A[8]); C[4] = det2x2_2(A[0], A[8], A[2], A[6]); C[5] = det2x2_2(A[1], A[6], A[0], A[7]);
  C[6] = det2x2_2(A[1], A[5], A[2], A[4]); C[7] = det2x2_2(A[2], A[3], A[0], A[5]); C[8] = det2x2_2(A[0], A[4], A[1], A[3]);
}
// Axis-aligned cell, tets j = 2m and 2m+1 as one packed pair: both run 0 -> s1 -> s2 -> 7 with
// the same first step (corner bit q0 = m, so column q0 of G is shared) and the other two steps
// swapped (q1 of one tet is q2 of the other), so every column position of the pair's G is a
// scaled difference of two corner rows per tet.
template <int m>
__device__ __forceinline__ void aa_pair_cols(const float (*u)[3], const float* inv, float2* G) {
  constexpr int jA = 2 * m, jB = 2 * m + 1;
  constexpr int s1 = CELL_TET(jA, 1), sA = CELL_TET(jA, 2), sB = CELL_TET(jB, 2);
  constexpr int q0 = CELL_Q(jA, 0), qa = CELL_Q(jA, 1), qb = CELL_Q(jA, 2);  // tet B: q1 = qb, q2 = qa
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const float c0 = (u[s1][r] - u[0][r]) * inv[q0];
    G[3 * r + q0] = make_float2(c0, c0);
    G[3 * r + qa] = mul2(make_float2(u[sA][r] - u[s1][r], u[7][r] - u[sB][r]), f2(inv[qa]));
    G[3 * r + qb] = mul2(make_float2(u[7][r] - u[sA][r], u[sB][r] - u[s1][r]), f2(inv[qb]));
  }
}
// gradient of a packed tet pair: energy (per tet, without the factor w = h^2 V), and the
// columns of P(F) and cof F scaled by 1/s_a (Pt[a][i] = w P_ia / s_a, Ct[a][i] = cof F_ia / s_a),
// whose path differences are the corner forces and cofactor vectors (see aa branch below)
__device__ __forceinline__ float2 grad_pair(const float2* Gm, float mu, float l2, float w, const float* inv, const float* invc,
                                           float2 (*Pt)[3], float2 (*Ct)[3]) {
  const float2 trG = add2(add2(Gm[0], Gm[4]), Gm[8]);
  const float2 i2 = add2(add2(det2x2_2(Gm[0], Gm[4], Gm[1], Gm[3]), det2x2_2(Gm[0], Gm[8], Gm[2], Gm[6])),
                         det2x2_2(Gm[4], Gm[8], Gm[5], Gm[7]));
  float2 cG[9];
  cof33_2(Gm, cG);
  const float2 detG = fma2(Gm[2], cG[2], fma2(Gm[1], cG[1], mul2(Gm[0], cG[0])));
  const float2 Jm1 = add2(add2(trG, i2), detG);
  float2 GG = mul2(Gm[0], Gm[0]);
#pragma unroll
  for (int i = 1; i < 9; ++i) GG = fma2(Gm[i], Gm[i], GG);
  // mu (GG/2 - i2 - detG) + l2/2 Jm1^2
  const float2 psi = fma2(mul2(f2(0.5f * l2), Jm1), Jm1, mul2(f2(mu), sub2(sub2(mul2(f2(0.5f), GG), i2), detG)));
  const float2 tr1 = add2(trG, f2(1.f));
  const float2 lj = mul2(f2(l2), Jm1);
  const float wmu = w * mu;
  const float2 wlj = mul2(f2(w), lj);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      // cof F = (1 + trG) I - G^T + cof G;  P(F) = mu (G + G^T - trG I - cof G) + lambda'(J-1) cof F
      const float2 cF = i == a ? add2(sub2(tr1, Gm[3 * a + i]), cG[3 * i + a]) : sub2(cG[3 * i + a], Gm[3 * a + i]);
      float2 sym = add2(Gm[3 * i + a], Gm[3 * a + i]);
      if (i == a) sym = sub2(sym, trG);
      const float2 PK = fma2(wlj, cF, mul2(f2(wmu), sub2(sym, cG[3 * i + a])));
      Pt[a][i] = mul2(PK, f2(inv[a]));
      Ct[a][i] = mul2(cF, f2(invc[a]));  // invc = inv sqrt(lambda' h^2 V): the blocks need no further scale
    }
  return psi;
}
// p^T H_e p of a packed tet pair (App. B quadratic form, as in the scalar loop below), per tet
// (without the common h^2 V factor)
__device__ __forceinline__ float2 curv_pair(const float2* Gm, const float2* dF, float mu, float l2) {
  const float2 trG = add2(add2(Gm[0], Gm[4]), Gm[8]);
  const float2 i2 = add2(add2(det2x2_2(Gm[0], Gm[4], Gm[1], Gm[3]), det2x2_2(Gm[0], Gm[8], Gm[2], Gm[6])),
                         det2x2_2(Gm[4], Gm[8], Gm[5], Gm[7]));
  float2 cG[9], cd[9];
  cof33_2(Gm, cG);
  cof33_2(dF, cd);
  const float2 detG = fma2(Gm[2], cG[2], fma2(Gm[1], cG[1], mul2(Gm[0], cG[0])));
  const float2 Jm1 = add2(add2(trG, i2), detG);
  const float2 tr1 = add2(trG, f2(1.f));
  float2 dd = f2(0.f), cfd = f2(0.f), fcd = f2(0.f);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) {
      const float2 cF = i == jj ? add2(sub2(tr1, Gm[3 * jj + i]), cG[3 * i + jj]) : sub2(cG[3 * i + jj], Gm[3 * jj + i]);
      const float2 Fij = i == jj ? add2(Gm[3 * i + jj], f2(1.f)) : Gm[3 * i + jj];
      dd = fma2(dF[3 * i + jj], dF[3 * i + jj], dd);
      cfd = fma2(cF, dF[3 * i + jj], cfd);
      fcd = fma2(Fij, cd[3 * i + jj], fcd);
    }
  // mu dd + l2 cfd^2 + 2 (l2 Jm1 - mu) fcd
  const float2 c2 = mul2(fma2(f2(l2), Jm1, f2(-mu)), f2(2.f));
  return fma2(c2, fcd, fma2(mul2(f2(l2), cfd), cfd, mul2(f2(mu), dd)));
}

// Axis-aligned cells (structured pads: corner bit b along axis b, signed edge s_b): column
// q_i of G is the scaled difference (u_{c_{i+1}} - u_{c_i}) / s_{q_i} along the path, and the
// b rows are e_q0/s_q0 - e_q1/s_q1, e_q1/s_q1 - e_q2/s_q2, e_q2/s_q2, so the corner forces and
// cofactor vectors are differences of scaled columns -- the same quantities with no 3x3
// products against stored b rows (cell_aa.w = tet volume > 0 marks such a cell)

// one packed pair of an axis-aligned cell: forces and lambda' c c^T blocks of both tets into the
// cell's corner accumulators.  Tet A (.x) runs 0 -> s1 -> sA -> 7 over columns q0, qa, qb, tet B
// (.y) 0 -> s1 -> sB -> 7 over q0, qb, qa; corner k of a path gets column(k-1) - column(k).
// (c arrives scaled by sqrt(lambda' h^2 V), so lambda' h^2 V c c^T is c c^T)
__device__ __forceinline__ void corner_acc(float* ag, float* aD, float f0, float f1, float f2_,
                                           float c0, float c1, float c2) {
  ag[0] += f0; ag[1] += f1; ag[2] += f2_;
  aD[0] = fmaf(c0, c0, aD[0]); aD[1] = fmaf(c1, c1, aD[1]); aD[2] = fmaf(c2, c2, aD[2]);
  aD[3] = fmaf(c0, c1, aD[3]); aD[4] = fmaf(c0, c2, aD[4]); aD[5] = fmaf(c1, c2, aD[5]);
}
template <int m>
__device__ __forceinline__ void pair_grad_acc(const float (*u)[3], const float* inv, const float* invc, float mu,
                                              float l2, float w, double& esum, float (*ag)[3], float (*aD)[6]) {
  constexpr int jA = 2 * m, jB = 2 * m + 1;
  constexpr int s1 = CELL_TET(jA, 1), sA = CELL_TET(jA, 2), sB = CELL_TET(jB, 2);
  constexpr int q0 = CELL_Q(jA, 0), qa = CELL_Q(jA, 1), qb = CELL_Q(jA, 2);
  float2 Gm[9], Pt[3][3], Ct[3][3];
  aa_pair_cols<m>(u, inv, Gm);
  const float2 psi = grad_pair(Gm, mu, l2, w, inv, invc, Pt, Ct);
  esum += (double)(w * psi.x);
  esum += (double)(w * psi.y);
  // tet A
  corner_acc(ag[0], aD[0], -Pt[q0][0].x, -Pt[q0][1].x, -Pt[q0][2].x, -Ct[q0][0].x, -Ct[q0][1].x, -Ct[q0][2].x);
  corner_acc(ag[s1], aD[s1], Pt[q0][0].x - Pt[qa][0].x, Pt[q0][1].x - Pt[qa][1].x, Pt[q0][2].x - Pt[qa][2].x,
             Ct[q0][0].x - Ct[qa][0].x, Ct[q0][1].x - Ct[qa][1].x, Ct[q0][2].x - Ct[qa][2].x);
  corner_acc(ag[sA], aD[sA], Pt[qa][0].x - Pt[qb][0].x, Pt[qa][1].x - Pt[qb][1].x, Pt[qa][2].x - Pt[qb][2].x,
             Ct[qa][0].x - Ct[qb][0].x, Ct[qa][1].x - Ct[qb][1].x, Ct[qa][2].x - Ct[qb][2].x);
  corner_acc(ag[7], aD[7], Pt[qb][0].x, Pt[qb][1].x, Pt[qb][2].x, Ct[qb][0].x, Ct[qb][1].x, Ct[qb][2].x);
  // tet B
  corner_acc(ag[0], aD[0], -Pt[q0][0].y, -Pt[q0][1].y, -Pt[q0][2].y, -Ct[q0][0].y, -Ct[q0][1].y, -Ct[q0][2].y);
  corner_acc(ag[s1], aD[s1], Pt[q0][0].y - Pt[qb][0].y, Pt[q0][1].y - Pt[qb][1].y, Pt[q0][2].y - Pt[qb][2].y,
             Ct[q0][0].y - Ct[qb][0].y, Ct[q0][1].y - Ct[qb][1].y, Ct[q0][2].y - Ct[qb][2].y);
  corner_acc(ag[sB], aD[sB], Pt[qb][0].y - Pt[qa][0].y, Pt[qb][1].y - Pt[qa][1].y, Pt[qb][2].y - Pt[qa][2].y,
             Ct[qb][0].y - Ct[qa][0].y, Ct[qb][1].y - Ct[qa][1].y, Ct[qb][2].y - Ct[qa][2].y);
  corner_acc(ag[7], aD[7], Pt[qa][0].y, Pt[qa][1].y, Pt[qa][2].y, Ct[qa][0].y, Ct[qa][1].y, Ct[qa][2].y);
}

// ALL_AA: every cell of the mesh is axis-aligned (structured pads) -- the stored-B branch is
// compiled out, which frees the registers it would hold
template <bool ALL_AA>
__global__ void __launch_bounds__(256, 2) k_elem_grad_cells(Dev d, float h2) {
  TAC_PDL_WAIT();
  int grp, bx, nbx;
  if (!group_block(d, (d.ncells + 7) / 8, blockIdx.y, blockIdx.x, gridDim.x, grp, bx, nbx)) return;
  const int e = grp * 32 + threadIdx.x;
  const bool act = e < d.E && (d.run[e] & 1);
  if (!__any_sync(0xffffffffu, act)) return;
  const float mu = d.emat[e], l2 = d.emat[d.Es + e];  // per-env material
  const unsigned G = (unsigned)(d.Es >> 5), eg = (unsigned)grp, lane = threadIdx.x;
  double esum = 0;
  for (int cidx = bx * 8 + threadIdx.y; cidx < d.ncells; cidx += nbx * 8) {
    const int4 va = __ldg(d.cell_v + 2 * cidx), vb4 = __ldg(d.cell_v + 2 * cidx + 1);
    const unsigned fix = __ldg(d.cell_fix + cidx);
    const float4 caa = __ldg(d.cell_aa + cidx);
    const bool aa = ALL_AA || caa.w > 0.f;  // warp-uniform (one cell per warp)
    const float inv[3] = {caa.x, caa.y, caa.z};
    if (!act) continue;
    const unsigned vb[8] = {(unsigned)va.x * G + eg, (unsigned)va.y * G + eg, (unsigned)va.z * G + eg,
                            (unsigned)va.w * G + eg, (unsigned)vb4.x * G + eg, (unsigned)vb4.y * G + eg,
                            (unsigned)vb4.z * G + eg, (unsigned)vb4.w * G + eg};
    float u[8][3];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const float* p = d.u + (vb[s] * 3u * 32u + lane);
#pragma unroll
      for (int c = 0; c < 3; ++c) u[s][c] = p[32 * c];
    }
    float ag[8][3], aD[8][6];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
      for (int c = 0; c < 3; ++c) ag[s][c] = 0.f;
#pragma unroll
      for (int c = 0; c < 6; ++c) aD[s][c] = 0.f;
    }
    // coalesced red.add of corner s's 9 accumulated terms (skipped for a fixed corner)
    auto flush = [&](int s) {
      if (fix & (1u << s)) return;
      float* pg = d.g + (vb[s] * 3u * 32u + lane);
      float* pd = d.D + (vb[s] * 6u * 32u + lane);
#pragma unroll
      for (int c = 0; c < 3; ++c) atomicAdd(pg + 32 * c, ag[s][c]);
#pragma unroll
      for (int c = 0; c < 6; ++c) atomicAdd(pd + 32 * c, aD[s][c]);
    };
    if constexpr (ALL_AA) {  // packed tet pairs (0,1), (2,3), (4,5); every tet has volume caa.w
      // each corner is flushed right after the last pair touching it (pair 0: corners 0 1 3 5 7,
      // pair 1: 0 2 3 6 7, pair 2: 0 4 5 6 7), so at most 6 corners' accumulators are live
      const float w = h2 * caa.w, sl = sqrtf(w * l2);
      const float invc[3] = {inv[0] * sl, inv[1] * sl, inv[2] * sl};
      pair_grad_acc<0>(u, inv, invc, mu, l2, w, esum, ag, aD);
      flush(1);
      pair_grad_acc<1>(u, inv, invc, mu, l2, w, esum, ag, aD);
      flush(2);
      flush(3);
      pair_grad_acc<2>(u, inv, invc, mu, l2, w, esum, ag, aD);
#pragma unroll
      for (int s : {0, 4, 5, 6, 7}) flush(s);
    } else {
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const int s0 = CELL_TET(j, 0), s1 = CELL_TET(j, 1), s2 = CELL_TET(j, 2), s3 = CELL_TET(j, 3);
      const int q0 = CELL_Q(j, 0), q1 = CELL_Q(j, 1), q2 = CELL_Q(j, 2);
      float Gm[9], b[3][3], vol;
      if (aa) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          Gm[3 * r + q0] = (u[s1][r] - u[s0][r]) * inv[q0];
          Gm[3 * r + q1] = (u[s2][r] - u[s1][r]) * inv[q1];
          Gm[3 * r + q2] = (u[s3][r] - u[s2][r]) * inv[q2];
        }
        vol = caa.w;
      } else {
        const float4 r0 = __ldg(d.cell_tb + 18 * cidx + 3 * j), r1 = __ldg(d.cell_tb + 18 * cidx + 3 * j + 1),
                     r2 = __ldg(d.cell_tb + 18 * cidx + 3 * j + 2);
        b[0][0] = r0.x; b[0][1] = r0.y; b[0][2] = r0.z;
        b[1][0] = r1.x; b[1][1] = r1.y; b[1][2] = r1.z;
        b[2][0] = r2.x; b[2][1] = r2.y; b[2][2] = r2.z;
        vol = r0.w;
        float du[3][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          du[0][c] = u[s1][c] - u[s0][c];
          du[1][c] = u[s2][c] - u[s0][c];
          du[2][c] = u[s3][c] - u[s0][c];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int jj = 0; jj < 3; ++jj) Gm[3 * i + jj] = du[0][i] * b[0][jj] + du[1][i] * b[1][jj] + du[2][i] * b[2][jj];
      }
      float trG = Gm[0] + Gm[4] + Gm[8];
      float i2 = (Gm[0] * Gm[4] - Gm[1] * Gm[3]) + (Gm[0] * Gm[8] - Gm[2] * Gm[6]) + (Gm[4] * Gm[8] - Gm[5] * Gm[7]);
      float cG[9];
      cof33(Gm, cG);
      float detG = Gm[0] * cG[0] + Gm[1] * cG[1] + Gm[2] * cG[2];
      float Jm1 = trG + i2 + detG;
      float GG = 0.f;
#pragma unroll
      for (int i = 0; i < 9; ++i) GG = fmaf(Gm[i], Gm[i], GG);
      float w = h2 * vol;
      esum += (double)(w * (mu * (0.5f * GG - i2 - detG) + 0.5f * l2 * Jm1 * Jm1));
      float cF[9], PK[9];
      const float lj = l2 * Jm1;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          cF[3 * i + jj] = (i == jj ? 1.f + trG : 0.f) - Gm[3 * jj + i] + cG[3 * i + jj];
          PK[3 * i + jj] = w * (mu * (Gm[3 * i + jj] + Gm[3 * jj + i] - (i == jj ? trG : 0.f) - cG[3 * i + jj]) + lj * cF[3 * i + jj]);
        }
      const float lc = w * l2;
      if (aa) {  // corner c: force and cofactor vector = differences of scaled columns
        float Pt[3][3], Ct[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int i = 0; i < 3; ++i) { Pt[a][i] = PK[3 * i + a] * inv[a]; Ct[a][i] = cF[3 * i + a] * inv[a]; }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int sk = k == 0 ? s0 : (k == 1 ? s1 : (k == 2 ? s2 : s3));
          float fv[3], cv[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            if (k == 0) { fv[i] = -Pt[q0][i]; cv[i] = -Ct[q0][i]; }
            else if (k == 1) { fv[i] = Pt[q0][i] - Pt[q1][i]; cv[i] = Ct[q0][i] - Ct[q1][i]; }
            else if (k == 2) { fv[i] = Pt[q1][i] - Pt[q2][i]; cv[i] = Ct[q1][i] - Ct[q2][i]; }
            else { fv[i] = Pt[q2][i]; cv[i] = Ct[q2][i]; }
            ag[sk][i] += fv[i];
          }
          aD[sk][0] += lc * cv[0] * cv[0]; aD[sk][1] += lc * cv[1] * cv[1]; aD[sk][2] += lc * cv[2] * cv[2];
          aD[sk][3] += lc * cv[0] * cv[1]; aD[sk][4] += lc * cv[0] * cv[2]; aD[sk][5] += lc * cv[1] * cv[2];
        }
      } else {
        float f0[3] = {0.f, 0.f, 0.f}, c0[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const int sk = kk == 0 ? s1 : (kk == 1 ? s2 : s3);
          float fv[3], cv[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            fv[i] = PK[3 * i] * b[kk][0] + PK[3 * i + 1] * b[kk][1] + PK[3 * i + 2] * b[kk][2];
            cv[i] = cF[3 * i] * b[kk][0] + cF[3 * i + 1] * b[kk][1] + cF[3 * i + 2] * b[kk][2];
            f0[i] -= fv[i];
            c0[i] -= cv[i];
            ag[sk][i] += fv[i];
          }
          aD[sk][0] += lc * cv[0] * cv[0]; aD[sk][1] += lc * cv[1] * cv[1]; aD[sk][2] += lc * cv[2] * cv[2];
          aD[sk][3] += lc * cv[0] * cv[1]; aD[sk][4] += lc * cv[0] * cv[2]; aD[sk][5] += lc * cv[1] * cv[2];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) ag[s0][i] += f0[i];
        aD[s0][0] += lc * c0[0] * c0[0]; aD[s0][1] += lc * c0[1] * c0[1]; aD[s0][2] += lc * c0[2] * c0[2];
        aD[s0][3] += lc * c0[0] * c0[1]; aD[s0][4] += lc * c0[0] * c0[2]; aD[s0][5] += lc * c0[1] * c0[2];
      }
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) flush(s);
    }
  }
  if (act) atomicAdd(d.acc + (size_t)A_EEL * d.Es + e, esum);
}

// ---- row-marching Kuhn-cell gradient (all cells axis-aligned): one warp = one segment of
// consecutive cells along corner bit 0 x 32 envs.  Cell k+1's corners 0, 2, 4, 6 are cell k's
// 1, 3, 5, 7, so their u and their force / block accumulators stay in registers from one cell
// to the next: per cell 12 corner row loads and 36 red.adds instead of 24 and 72.  Pair order
// 1, 2, 0 finishes the carried-in corners early (2 after pair 1; 4, 6 after pair 2; 0 after
// pair 0), so at most 6 corners' accumulators are live, as in the one-cell pass.
constexpr int kRowWarps = 6;  // warps per CTA of the row-marching gradient
template <bool TOL>
__global__ void __launch_bounds__(32 * kRowWarps, 2) k_elem_grad_rows(Dev d, float h2) {
  TAC_PDL_WAIT();
  int e, bx, nbx;
  if (!env_lanes<TOL>(d, (d.nseg + kRowWarps - 1) / kRowWarps, blockIdx.y, blockIdx.x, gridDim.x, e, bx, nbx)) return;
  const bool act = e < d.E && (d.run[e] & 1);
  if (!__any_sync(0xffffffffu, act)) return;
  const float mu = d.emat[e], l2 = d.emat[d.Es + e];  // per-env material
  const unsigned G = (unsigned)(d.Es >> 5), eg = TOL ? (unsigned)e >> 5 : (unsigned)blockIdx.y,
                 lane = TOL ? (unsigned)e & 31u : (unsigned)threadIdx.x;  // (compacted: per lane)
  double esum = 0;
  // the segment's cell records (corner ids, fixed mask, axis-aligned box) staged per warp in
  // shared memory at the segment start: one load round trip per segment instead of one per cell
  // (the corner-row address arithmetic waited on each cell's record)
  __shared__ int4 smv[kRowWarps][2 * kRowSegMax];
  __shared__ float4 sma[kRowWarps][kRowSegMax];
  __shared__ unsigned smf[kRowWarps][kRowSegMax];
  const int ty = threadIdx.y, tl = threadIdx.x;
  for (int sg = bx * kRowWarps + threadIdx.y; sg < d.nseg; sg += nbx * kRowWarps) {
    const int2 seg = __ldg(d.cell_seg + sg);
    if (tl < 2 * seg.y) smv[ty][tl] = __ldg(d.cell_v + 2 * seg.x + tl);
    if (tl < seg.y) { smf[ty][tl] = __ldg(d.cell_fix + seg.x + tl); sma[ty][tl] = __ldg(d.cell_aa + seg.x + tl); }
    __syncwarp();
    if (act) {
    float u[8][3], ag[8][3], aD[8][6];
    {  // the first cell's -x face into the slots of the +x face (shifted in below)
      const int4 va = smv[ty][0], vb4 = smv[ty][1];
      const unsigned f[4] = {(unsigned)va.x, (unsigned)va.z, (unsigned)vb4.x, (unsigned)vb4.z};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float* p = d.u + ((f[k] * G + eg) * 3u * 32u + lane);
#pragma unroll
        for (int c = 0; c < 3; ++c) { u[2 * k + 1][c] = p[32 * c]; ag[2 * k + 1][c] = 0.f; }
#pragma unroll
        for (int c = 0; c < 6; ++c) aD[2 * k + 1][c] = 0.f;
      }
    }
    for (int ci = 0; ci < seg.y; ++ci) {
      const int4 va = smv[ty][2 * ci], vb4 = smv[ty][2 * ci + 1];
      const unsigned fix = smf[ty][ci];
      const float4 caa = sma[ty][ci];
      const float inv[3] = {caa.x, caa.y, caa.z};
      const unsigned vb[8] = {(unsigned)va.x * G + eg, (unsigned)va.y * G + eg, (unsigned)va.z * G + eg,
                              (unsigned)va.w * G + eg, (unsigned)vb4.x * G + eg, (unsigned)vb4.y * G + eg,
                              (unsigned)vb4.z * G + eg, (unsigned)vb4.w * G + eg};
      // shift the previous cell's +x face into this cell's -x face, load the new +x face
      // (loading rows 1 and 5 just before their first pair measured 187.8 vs 184.6 us)
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { u[k][c] = u[k + 1][c]; ag[k][c] = ag[k + 1][c]; ag[k + 1][c] = 0.f; }
#pragma unroll
        for (int c = 0; c < 6; ++c) { aD[k][c] = aD[k + 1][c]; aD[k + 1][c] = 0.f; }
        const float* p = d.u + (vb[k + 1] * 3u * 32u + lane);
#pragma unroll
        for (int c = 0; c < 3; ++c) u[k + 1][c] = p[32 * c];
      }
      auto flush = [&](int s) {
        if (fix & (1u << s)) return;
        float* pg = d.g + (vb[s] * 3u * 32u + lane);
        float* pd = d.D + (vb[s] * 6u * 32u + lane);
#pragma unroll
        for (int c = 0; c < 3; ++c) atomicAdd(pg + 32 * c, ag[s][c]);
#pragma unroll
        for (int c = 0; c < 6; ++c) atomicAdd(pd + 32 * c, aD[s][c]);
      };
      const float w = h2 * caa.w, sl = sqrtf(w * l2);
      const float invc[3] = {inv[0] * sl, inv[1] * sl, inv[2] * sl};
      pair_grad_acc<1>(u, inv, invc, mu, l2, w, esum, ag, aD);  // corners 0 2 3 6 7
      flush(2);
      pair_grad_acc<2>(u, inv, invc, mu, l2, w, esum, ag, aD);  // corners 0 4 5 6 7
      flush(4);
      flush(6);
      pair_grad_acc<0>(u, inv, invc, mu, l2, w, esum, ag, aD);  // corners 0 1 3 5 7
      flush(0);
      if (ci == seg.y - 1) {
        flush(1);
        flush(3);
        flush(5);
        flush(7);
      }
    }
    }  // act
    __syncwarp();  // the records are read before the next segment's staging overwrites them
  }
  if (act) atomicAdd(d.acc + (size_t)A_EEL * d.Es + e, esum);
}

// ------------------------------------------------------------------ a7: curvature
// p^T H_e p = h^2 V [mu |dF|^2 + lambda' (cof F : dF)^2 + 2 (lambda'(J-1) - mu) F : cof(dF)]  (App. B)

// ---- Kuhn-cell element curvature: one warp = one cell x 32 envs, u and p of the 8 corners
// in registers; p^T H_e p summed over the 6 tets (App. B quadratic form)
template <bool ALL_AA, bool TOL>
__global__ void __launch_bounds__(256, 2) k_elem_curv_cells(Dev d, float h2) {
  TAC_PDL_WAIT();
  int e, bx, nbx;
  if (!env_lanes<TOL>(d, (d.ncells + 7) / 8, blockIdx.y, blockIdx.x, gridDim.x, e, bx, nbx)) return;
  const bool act = e < d.E && (d.run[e] & 2);
  if (!__any_sync(0xffffffffu, act)) return;
  const float mu = d.emat[e], l2 = d.emat[d.Es + e];  // per-env material
  const unsigned G = (unsigned)(d.Es >> 5), eg = TOL ? (unsigned)e >> 5 : (unsigned)blockIdx.y,
                 lane = TOL ? (unsigned)e & 31u : (unsigned)threadIdx.x;  // (compacted: per lane)
  double qsum = 0;
  // the next cell's record is loaded ahead (the corner-row addresses wait on it)
  const int cstep = nbx * 8;
  int4 nva = make_int4(0, 0, 0, 0), nvb = make_int4(0, 0, 0, 0);
  float4 ncaa = make_float4(0.f, 0.f, 0.f, 0.f);
  if (bx * 8 + (int)threadIdx.y < d.ncells) {
    const int c0 = bx * 8 + threadIdx.y;
    nva = __ldg(d.cell_v + 2 * c0); nvb = __ldg(d.cell_v + 2 * c0 + 1); ncaa = __ldg(d.cell_aa + c0);
  }
  for (int cidx = bx * 8 + threadIdx.y; cidx < d.ncells; cidx += cstep) {
    const int4 va = nva, vb4 = nvb;
    const float4 caa = ncaa;
    if (cidx + cstep < d.ncells) {
      nva = __ldg(d.cell_v + 2 * (cidx + cstep)); nvb = __ldg(d.cell_v + 2 * (cidx + cstep) + 1);
      ncaa = __ldg(d.cell_aa + cidx + cstep);
    }
    const bool aa = ALL_AA || caa.w > 0.f;  // warp-uniform (one cell per warp)
    const float inv[3] = {caa.x, caa.y, caa.z};
    if (!act) continue;
    const unsigned vb[8] = {(unsigned)va.x * G + eg, (unsigned)va.y * G + eg, (unsigned)va.z * G + eg,
                            (unsigned)va.w * G + eg, (unsigned)vb4.x * G + eg, (unsigned)vb4.y * G + eg,
                            (unsigned)vb4.z * G + eg, (unsigned)vb4.w * G + eg};
    float u[8][3], p[8][3];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const float* pu = d.u + (vb[s] * 3u * 32u + lane);
      const float* pp = d.p + (vb[s] * 3u * 32u + lane);
#pragma unroll
      for (int c = 0; c < 3; ++c) { u[s][c] = pu[32 * c]; p[s][c] = pp[32 * c]; }
    }
    float q = 0.f;
    if constexpr (ALL_AA) {  // packed tet pairs (0,1), (2,3), (4,5); every tet has volume caa.w
      float2 qp = f2(0.f);
      {
        float2 Gm[9], dF[9];
        aa_pair_cols<0>(u, inv, Gm);
        aa_pair_cols<0>(p, inv, dF);
        qp = add2(qp, curv_pair(Gm, dF, mu, l2));
      }
      {
        float2 Gm[9], dF[9];
        aa_pair_cols<1>(u, inv, Gm);
        aa_pair_cols<1>(p, inv, dF);
        qp = add2(qp, curv_pair(Gm, dF, mu, l2));
      }
      {
        float2 Gm[9], dF[9];
        aa_pair_cols<2>(u, inv, Gm);
        aa_pair_cols<2>(p, inv, dF);
        qp = add2(qp, curv_pair(Gm, dF, mu, l2));
      }
      qsum += (double)(h2 * (caa.w * (qp.x + qp.y)));
    } else {
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const int s0 = CELL_TET(j, 0), s1 = CELL_TET(j, 1), s2 = CELL_TET(j, 2), s3 = CELL_TET(j, 3);
      const int q0 = CELL_Q(j, 0), q1 = CELL_Q(j, 1), q2 = CELL_Q(j, 2);
      float Gm[9], dF[9], vol;
      if (aa) {  // axis-aligned cell: scaled differences along the path (see CELL_Q)
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          Gm[3 * r + q0] = (u[s1][r] - u[s0][r]) * inv[q0];
          Gm[3 * r + q1] = (u[s2][r] - u[s1][r]) * inv[q1];
          Gm[3 * r + q2] = (u[s3][r] - u[s2][r]) * inv[q2];
          dF[3 * r + q0] = (p[s1][r] - p[s0][r]) * inv[q0];
          dF[3 * r + q1] = (p[s2][r] - p[s1][r]) * inv[q1];
          dF[3 * r + q2] = (p[s3][r] - p[s2][r]) * inv[q2];
        }
        vol = caa.w;
      } else {
        const float4 r0 = __ldg(d.cell_tb + 18 * cidx + 3 * j), r1 = __ldg(d.cell_tb + 18 * cidx + 3 * j + 1),
                     r2 = __ldg(d.cell_tb + 18 * cidx + 3 * j + 2);
        const float b[3][3] = {{r0.x, r0.y, r0.z}, {r1.x, r1.y, r1.z}, {r2.x, r2.y, r2.z}};
        vol = r0.w;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const float du0 = u[s1][i] - u[s0][i], du1 = u[s2][i] - u[s0][i], du2 = u[s3][i] - u[s0][i];
          const float dp0 = p[s1][i] - p[s0][i], dp1 = p[s2][i] - p[s0][i], dp2 = p[s3][i] - p[s0][i];
#pragma unroll
          for (int jj = 0; jj < 3; ++jj) {
            Gm[3 * i + jj] = du0 * b[0][jj] + du1 * b[1][jj] + du2 * b[2][jj];
            dF[3 * i + jj] = dp0 * b[0][jj] + dp1 * b[1][jj] + dp2 * b[2][jj];
          }
        }
      }
      float trG = Gm[0] + Gm[4] + Gm[8];
      float i2 = (Gm[0] * Gm[4] - Gm[1] * Gm[3]) + (Gm[0] * Gm[8] - Gm[2] * Gm[6]) + (Gm[4] * Gm[8] - Gm[5] * Gm[7]);
      float cG[9], cd[9];
      cof33(Gm, cG);
      cof33(dF, cd);
      float detG = Gm[0] * cG[0] + Gm[1] * cG[1] + Gm[2] * cG[2];
      float Jm1 = trG + i2 + detG;
      float dd = 0.f, cfd = 0.f, fcd = 0.f;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          float cF = (i == jj ? 1.f + trG : 0.f) - Gm[3 * jj + i] + cG[3 * i + jj];
          float Fij = (i == jj ? 1.f : 0.f) + Gm[3 * i + jj];
          dd = fmaf(dF[3 * i + jj], dF[3 * i + jj], dd);
          cfd = fmaf(cF, dF[3 * i + jj], cfd);
          fcd = fmaf(Fij, cd[3 * i + jj], fcd);
        }
      q += vol * (mu * dd + l2 * cfd * cfd + 2.f * (l2 * Jm1 - mu) * fcd);
    }
    qsum += (double)(h2 * q);
    }
  }
  if (act) atomicAdd(d.acc + (size_t)A_PHP * d.Es + e, qsum);
}

// ---- tiled element passes: one CTA = one tile x 32 envs (lane = env) ----
// Vertex rows of the tile are staged in shared memory once (instead of once per tet);
// gradient and diagonal blocks accumulate in shared memory in rounds of vertex-disjoint
// tets (one per warp, no atomics), and each tile vertex is flushed once: plain
// read-modify-write if only this tile touches it, a coalesced red.add otherwise.
__device__ __forceinline__ TetData load_tile_tet(const Dev& d, int gt) {
  TetData T;
  float4 r0 = __ldg(d.tile_tb + 3 * gt), r1 = __ldg(d.tile_tb + 3 * gt + 1), r2 = __ldg(d.tile_tb + 3 * gt + 2);
  T.b[0][0] = r0.x; T.b[0][1] = r0.y; T.b[0][2] = r0.z; T.vol = r0.w;
  T.b[1][0] = r1.x; T.b[1][1] = r1.y; T.b[1][2] = r1.z;
  T.b[2][0] = r2.x; T.b[2][1] = r2.y; T.b[2][2] = r2.z;
  return T;
}
constexpr int kTiledCurvSmem = 2 * 3 * kTileV * 32 * 4;
__global__ void __launch_bounds__(256) k_elem_curv_tiled(Dev d, float h2) {
  TAC_PDL_WAIT();
  extern __shared__ float shc[];
  float (*su)[kTileV][32] = reinterpret_cast<float (*)[kTileV][32]>(shc);
  float (*sp)[kTileV][32] = reinterpret_cast<float (*)[kTileV][32]>(shc + 3 * kTileV * 32);
  __shared__ double se[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane, tile = blockIdx.y;
  const bool act = e < d.E && (d.run[e] & 2);
  if (!__syncthreads_or(act)) return;
  const int v0 = d.tile_vstart[tile], nvt = d.tile_vstart[tile + 1] - v0;
  for (int lv = w; lv < nvt; lv += 8) {
    int gv = d.tile_verts[v0 + lv];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      su[c][lv][lane] = act ? d.u[vidx(d, c, gv, e)] : 0.f;
      sp[c][lv][lane] = act ? d.p[vidx(d, c, gv, e)] : 0.f;
    }
  }
  __syncthreads();
  const float mu = d.emat[e], l2 = d.emat[d.Es + e];  // per-env material
  const int t0 = d.tile_tstart[tile], nt = d.tile_tstart[tile + 1] - t0;
  double qsum = 0;
  if (act) {
    for (int lt = w; lt < nt; lt += 8) {
      uchar4 tv = __ldg(d.tile_tv + t0 + lt);
      int lv4[4] = {tv.x, tv.y, tv.z, tv.w};
      TetData T = load_tile_tet(d, t0 + lt);
      float du[3][3], dp[3][3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          du[k][c] = su[c][lv4[k + 1]][lane] - su[c][lv4[0]][lane];
          dp[k][c] = sp[c][lv4[k + 1]][lane] - sp[c][lv4[0]][lane];
        }
      float G[9], dF[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          float s = 0.f, q = 0.f;
#pragma unroll
          for (int k = 0; k < 3; ++k) { s = fmaf(du[k][i], T.b[k][j], s); q = fmaf(dp[k][i], T.b[k][j], q); }
          G[3 * i + j] = s;
          dF[3 * i + j] = q;
        }
      float trG = G[0] + G[4] + G[8];
      float i2 = (G[0] * G[4] - G[1] * G[3]) + (G[0] * G[8] - G[2] * G[6]) + (G[4] * G[8] - G[5] * G[7]);
      float cG[9], cd[9];
      cof33(G, cG);
      cof33(dF, cd);
      float detG = G[0] * cG[0] + G[1] * cG[1] + G[2] * cG[2];
      float Jm1 = trG + i2 + detG;
      float dd = 0.f, cfd = 0.f, fcd = 0.f;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          float cF = (i == j ? 1.f + trG : 0.f) - G[3 * j + i] + cG[3 * i + j];
          float Fij = (i == j ? 1.f : 0.f) + G[3 * i + j];
          dd = fmaf(dF[3 * i + j], dF[3 * i + j], dd);
          cfd = fmaf(cF, dF[3 * i + j], cfd);
          fcd = fmaf(Fij, cd[3 * i + j], fcd);
        }
      qsum += (double)(h2 * T.vol * (mu * dd + l2 * cfd * cfd + 2.f * (l2 * Jm1 - mu) * fcd));
    }
  }
  se[w][lane] = qsum;
  __syncthreads();
  if (w == 0 && act) {
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += se[j][lane];
    atomicAdd(d.acc + (size_t)A_PHP * d.Es + e, s);
  }
}

// ------------------------------------------------------------------ a5: contact gradient
// barrier kappa b(d) over candidates with d < dhat, Gauss-Newton diagonal
// kappa b'' w_k^2 n n^T (R8); friction mu_f lambda f(|T^T Delta|) over anchors
// with GN diagonal mu lambda f1 w_k^2 T T^T; indenter corners reduce to the
// rigid wrench (g_c += f, g_theta += (y - c) x f).
__device__ __forceinline__ void add_sym(double* A, d3 a, double s) {  // A(6) += s a a^T
  A[0] += s * a.x * a.x; A[1] += s * a.y * a.y; A[2] += s * a.z * a.z;
  A[3] += s * a.x * a.y; A[4] += s * a.x * a.z; A[5] += s * a.y * a.z;
}
// v: free gel vertex id (gradient), sl: its surface-local id (contact block, Dcon)
__device__ __forceinline__ void scatter_gel_free(const Dev& d, int v, int sl, int e, d3 f, double s, d3 n) {
  atomicAdd(d.g + vidx(d, 0, v, e), (float)f.x);
  atomicAdd(d.g + vidx(d, 1, v, e), (float)f.y);
  atomicAdd(d.g + vidx(d, 2, v, e), (float)f.z);
  if (s != 0.0) {
    atomicAdd(d.Dcon + vidxS(d, 0, sl, e), (float)(s * n.x * n.x));
    atomicAdd(d.Dcon + vidxS(d, 1, sl, e), (float)(s * n.y * n.y));
    atomicAdd(d.Dcon + vidxS(d, 2, sl, e), (float)(s * n.z * n.z));
    atomicAdd(d.Dcon + vidxS(d, 3, sl, e), (float)(s * n.x * n.y));
    atomicAdd(d.Dcon + vidxS(d, 4, sl, e), (float)(s * n.x * n.z));
    atomicAdd(d.Dcon + vidxS(d, 5, sl, e), (float)(s * n.y * n.z));
  }
}


// ---- per-env contact grids: gridDim.x blocks per env x E.  In the tolerance mode, once few
// envs are still iterating (the tail of a step: n < remap_blocks / gridDim.x), the blocks are
// dealt over the envs of k_alpha's list (alist, the envs evaluating next) -- each gets up to
// min(kMaxEnvBlocks, remap_blocks / n) blocks, so a straggler's contact passes are not run by
// one CTA while the GPU idles.  With more envs active, without a list (fixed mode, the first
// evaluation of a step) the mapping is the identity (e = blockIdx.y, bx = blockIdx.x): splitting
// many envs over more CTAs only repeats per-CTA setup (measured, tools/diag_tail.py).  The
// curvature passes (bit 2) use the same list: their envs are a subset of the evaluated ones.
constexpr int kMaxEnvBlocks = 64;
__device__ __forceinline__ bool env_block(const Dev& d, int bit, int& e, int& bx, int& nbx) {
  bx = blockIdx.x;
  nbx = gridDim.x;
  if (d.fixed_iters <= 0 && (int)gridDim.x < kMaxEnvBlocks) {
    const int n = d.anum[0], T = gridDim.x * gridDim.y;  // (n * per <= T: every listed env gets all per blocks)
    const int per = n > 0 ? min(kMaxEnvBlocks, min(d.remap_blocks, T) / n) : 0;
    if (per > (int)gridDim.x) {
      const int lin = blockIdx.y * gridDim.x + blockIdx.x, idx = lin / per;
      if (idx >= n) return false;
      nbx = per;
      bx = lin - idx * per;
      e = d.alist[idx];
      return (d.run[e] & bit) != 0;
    }
  }
  e = blockIdx.y;
  return e < d.E && (d.run[e] & bit);
}

template <int KIND, bool MOLL = false>  // MOLL: edge-edge mollifier (R30), KIND 2 only
__global__ void __launch_bounds__(128) k_contact_near(Dev d, double h2) {
  TAC_PDL_WAIT();
  int e, bx, nbx;
  if (!env_block(d, 1, e, bx, nbx)) return;
  const double kappa = h2 * d.edbl[e];  // h^2 kappa_phys of this env
  const EnvS& s = d.es[e];
  __shared__ double R[9], c[3];
  __shared__ double smr[4 * 20];
  if (threadIdx.x < 9) R[threadIdx.x] = s.R[threadIdx.x];
  if (threadIdx.x < 3) c[threadIdx.x] = s.c[threadIdx.x];
  __syncthreads();
  double Eb = 0, gr[6] = {0, 0, 0, 0, 0, 0}, Dc[6] = {0, 0, 0, 0, 0, 0}, Dt[6] = {0, 0, 0, 0, 0, 0};
  d3 cc = ld3(c);
  const int n = d.nnear[3 * e + KIND];
  // near-ordered output slots: kinds 0, 1, 2 concatenated (the counts are final after classify)
  const int base = (KIND >= 1 ? d.nnear[3 * e] : 0) + (KIND >= 2 ? d.nnear[3 * e + 1] : 0);
  const uint2* list = d.nearl + ((size_t)e * 3 + KIND) * d.kmax;  // packed corners of the near pairs
  constexpr float kNearScreen = 1e-6f;
  const float far2 = ((float)d.dhat + kNearScreen) * ((float)d.dhat + kNearScreen);
  bool far = false;
  // the next round's corner word is loaded at the top of each round (one dependent round trip
  // less per pair: the corner gathers wait on it)
  const int jstep = nbx * blockDim.x;
  uint2 cw_next = make_uint2(0u, 0u);
  if (bx * blockDim.x + threadIdx.x < n) cw_next = list[bx * blockDim.x + threadIdx.x];
  for (int j = bx * blockDim.x + threadIdx.x; j < n; j += jstep) {
    const uint2 cw = cw_next;
    if (j + jstep < n) cw_next = list[j + jstep];
    const unsigned id[4] = {cw.x & 0xffffu, cw.x >> 16, cw.y & 0xffffu, (cw.y >> 16) & 0x3fffu};
    bool ind[4];
    d3 z[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ind[k] = KIND == 0 ? k >= 1 : (KIND == 1 ? k == 0 : k >= 2);
      if (ind[k]) {
        z[k] = mv(R, ind_body(d, id[k])) + cc;
      } else {
        const float4 X = __ldg(d.Xs + id[k]), u = d.usurf[(size_t)id[k] * d.Es + e];
        z[k] = mk((double)X.x + (double)u.x, (double)X.y + (double)u.y, (double)X.z + (double)u.z);
      }
    }
    const size_t slot = (size_t)e * d.kmax + base + j;
    d.ncorn[slot] = cw;
    float4* geo = d.cgeo + 2 * slot;
    if (KIND != 2) {  // fp32 screen (point-triangle kinds; edge-edge near pairs are nearly all
       // within dhat, measured: the screen cost more than it saved there): a pair at exact
       // distance >= dhat carries no energy and is covered by the shared far-pair step bound
       // (R15), like a pair the classification certified
      f3 zf[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) zf[k] = f3{(float)(z[k].x - z[0].x), (float)(z[k].y - z[0].y), (float)(z[k].z - z[0].z)};
      const float d2 = KIND == 2 ? dist2_ee_f(zf[0], zf[1], zf[2], zf[3]) : dist2_pt_f(zf[0], zf[1], zf[2], zf[3]);
      if (d2 >= far2) {
        far = true;
        geo[0] = make_float4(0.f, 0.f, 0.f, 0.f);  // skipped by the curvature pass
        continue;
      }
    }
    DR D = KIND == 2 ? dist_ee(z[0], z[1], z[2], z[3]) : dist_pt(z[0], z[1], z[2], z[3]);
    if (!(D.d > 0)) {
      Eb = INFINITY;
      geo[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      geo[1] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    if (D.d >= d.dhat) {  // exact distance >= dhat: far (R15), as the fp32 screen above
      far = true;
      geo[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    bool ee_int = true;
    if (d.dedup && dedup_duplicate(d, e, id, ind, D.w, &ee_int)) {  // R33: counted by another pair
      geo[0] = make_float4(0.f, 0.f, 0.f, 0.f);                     // (same geometry: nothing to add)
      continue;
    }
    d3 rr = mk(0, 0, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) rr = rr + D.w[k] * z[k];
    d3 nn = (1.0 / D.d) * rr;
    MollD Mo;
    Mo.m = 1.0;
    Mo.dm = 0.0;
    if (MOLL && ee_int)  // R30 (gel corners 0, 1 surface-local; indenter corners 2, 3); with R33 edge-edge only
      Mo = ee_moll(z, sqlen4(__ldg(d.Xs + id[1]), __ldg(d.Xs + id[0])), sqlen4(__ldg(d.Y + id[3]), __ldg(d.Y + id[2])));
    geo[0] = make_float4((float)D.d, (float)nn.x, (float)nn.y, (float)nn.z);
    const double sm = (MOLL && ee_int) ? sqrt(Mo.m) : 1.0;  // curvature weights carry sqrt(m): m kappa b'' (n . dr)^2
    geo[1] = make_float4((float)(sm * D.w[0]), (float)(sm * D.w[1]), (float)(sm * D.w[2]), (float)(sm * D.w[3]));
    double lg = log(D.d / d.dhat), dm = D.d - d.dhat, inv = 1.0 / D.d;
    const double bk = kappa * (-dm * dm * lg);                           // kappa b
    Eb += Mo.m * bk;
    double db = Mo.m * kappa * (-2 * dm * lg - dm * dm * inv);                  // m kappa b'
    double ddb = Mo.m * kappa * (-2 * lg - 4 * dm * inv + dm * dm * inv * inv); // m kappa b'' (GN)
    const double bdm = bk * Mo.dm;                                       // kappa b m' (R30)
    double sig = 0;
    d3 rho = mk(0, 0, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      d3 f = (db * D.w[k]) * nn;
      if (MOLL && ee_int) f = f + bdm * Mo.dc[k];
      if (!ind[k]) {
        const int v = __ldg(d.svfree + id[k]);  // one load: id and fixed flag
        if (v >= 0) scatter_gel_free(d, v, id[k], e, f, ddb * D.w[k] * D.w[k], nn);
      } else {
        d3 arm = z[k] - cc;
        d3 tq = cross(arm, f);
        gr[0] += f.x; gr[1] += f.y; gr[2] += f.z; gr[3] += tq.x; gr[4] += tq.y; gr[5] += tq.z;
        sig += D.w[k];
        rho = rho + D.w[k] * arm;
      }
    }
    add_sym(Dc, nn, ddb * sig * sig);
    add_sym(Dt, cross(rho, nn), ddb);
  }
  if (__any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0)
    atomic_min_pos(d.accu + (size_t)U_GFAR * d.Es + e, (float)d.dhat);
  double vals[20];
  vals[0] = Eb;
  vals[1] = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    vals[2 + k] = gr[k];
    vals[8 + k] = Dc[k];
    vals[14 + k] = Dt[k];
  }
  block_sums_contact(vals, d.acc, d.Es, e, smr);
}


// Run-based warp reduction of one gel vertex's 9 contact terms: maximal runs of equal
// adjacent keys (anchors are sorted per step, so an anchor's gel primitive repeats in
// neighbouring lanes) are summed by a log-step segmented scan and the run's last lane issues
// the red.add.  Correct for any order (non-adjacent duplicates form separate runs).
__device__ __forceinline__ void seg_red9(const Dev& d, int e, unsigned key, float* v) {
  const int lane = threadIdx.x & 31;
  const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1), next = __shfl_down_sync(0xffffffffu, key, 1);
  const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || prev != key);
  const int start = 31 - __clz(heads & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u)));
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const float t = __shfl_up_sync(0xffffffffu, v[k], off);
      if (lane - off >= start) v[k] += t;
    }
  }
  if (key == 0xffffffffu || (lane != 31 && next == key)) return;  // only the run's last lane
#pragma unroll
  for (int c = 0; c < 3; ++c) atomicAdd(d.g + vidx(d, c, key, e), v[c]);
  const int sl = __ldg(d.sidx + key);  // the contact block lives with the surface vertex
#pragma unroll
  for (int c = 0; c < 6; ++c) atomicAdd(d.Dcon + vidxS(d, c, sl, e), v[3 + c]);
}

// per-step anchor order: by (first, second) free gel corner, so anchors of one gel primitive
// sit in neighbouring lanes of the friction pass (seg_red9).  One CTA per env, bitonic sort
// of (key | index) in shared memory, then a gather into the second anchor buffer.
__global__ void __launch_bounds__(1024) k_sort_anchors(Dev d, Anchor* out) {
  TAC_PDL_WAIT();
  extern __shared__ unsigned long long skey[];
  const int e = blockIdx.x;
  if (d.es[e].mode != kActive) return;
  const int na = min(d.nanc[e], d.amax);
  int n = 1;
  while (n < na) n <<= 1;
  const Anchor* in = d.anc + (size_t)e * d.amax;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (i < na) {
      const unsigned long long g0 = (unsigned)(in[i].gid[0] + 1), g1 = (unsigned)(in[i].gid[1] + 1);
      skey[i] = (g0 << 42) | (g1 << 20) | (unsigned long long)i;
    } else {
      skey[i] = ~0ull;
    }
  }
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = skey[i], b = skey[l];
          if (((i & k) == 0) == (a > b)) { skey[i] = b; skey[l] = a; }
        }
      }
      __syncthreads();
    }
  Anchor* o = out + (size_t)e * d.amax;
  for (int i = threadIdx.x; i < na; i += blockDim.x) o[i] = in[skey[i] & 0xfffffull];
}

// friction over the anchors: value, gradient, GN blocks, wrench; caches
// mu lambda f1(s) per anchor for the curvature pass
__global__ void __launch_bounds__(128) k_contact_friction(Dev d, double eps_f) {
  TAC_PDL_WAIT();
  int e, bx, nbx;
  if (!env_block(d, 1, e, bx, nbx)) return;
  const EnvS& s = d.es[e];
  __shared__ double R[9], c[3];
  __shared__ double smr[4 * 20];
  if (threadIdx.x < 9) R[threadIdx.x] = s.R[threadIdx.x];
  if (threadIdx.x < 3) c[threadIdx.x] = s.c[threadIdx.x];
  __syncthreads();
  double Ef = 0, gr[6] = {0, 0, 0, 0, 0, 0}, Dc[6] = {0, 0, 0, 0, 0, 0}, Dt[6] = {0, 0, 0, 0, 0, 0};
  const d3 cc = ld3(c);
  const int na = min(d.nanc[e], d.amax);
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count (the aggregated scatter is a warp collective)
  for (int b0 = bx * blockDim.x + (threadIdx.x & ~31); b0 < na; b0 += nbx * blockDim.x) {
    const int i = b0 + lane;
    // per-corner terms are formed at their reduction from a few shared factors (force
    // direction, T T^T entries, f1 and the corner weights), not held as 3 x 9 values
    unsigned key[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu};
    float Ttf[3] = {0.f, 0.f, 0.f}, tt[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, wf[3] = {0.f, 0.f, 0.f};
    float f1f = 0.f;
    if (i < na) {
    // (loading the next round's corner ids ahead, as in the curvature pass, measured 95 -> 101 us
    // here: 144 instead of 128 registers)
    const Anchor& A = d.anc[(size_t)e * d.amax + i];
    const int gid[3] = {A.gid[0], A.gid[1], A.gid[2]};
    const unsigned sid[3] = {A.sid01 & 0xffffu, A.sid01 >> 16, A.sid2};
    float4 us[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)  // all corner loads in flight at once
      if (gid[k] >= 0) us[k] = d.usurf[(size_t)sid[k] * d.Es + e];
    const d3 rho = mv(R, mk(A.yw[0], A.yw[1], A.yw[2]));  // sum_ind w (y - c) = R Y_w
    const double sig = A.sig;
    d3 Dl = rho + sig * cc - mk(A.c0[0], A.c0[1], A.c0[2]);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (gid[k] >= 0) Dl = Dl + (double)A.w[k] * mk(us[k].x, us[k].y, us[k].z);
    d3 t1 = mk(A.t1[0], A.t1[1], A.t1[2]), t2 = mk(A.t2[0], A.t2[1], A.t2[2]);
    double ta = dot(t1, Dl), tb = dot(t2, Dl);
    double sn = sqrt(ta * ta + tb * tb);
    double ml = d.edbl[d.Es + e] * (double)A.lam;  // per-env mu_f
    Ef += ml * moll_f(sn, eps_f);
    double f1 = ml * moll_f1(sn, eps_f);
    d.anc_f1[(size_t)e * d.amax + i] = (float)f1;
    d3 Tt = ta * t1 + tb * t2;
    f1f = (float)f1;
    Ttf[0] = (float)Tt.x; Ttf[1] = (float)Tt.y; Ttf[2] = (float)Tt.z;
    // GN: f1 w^2 T T^T (R8)
    tt[0] = (float)(t1.x * t1.x + t2.x * t2.x); tt[1] = (float)(t1.y * t1.y + t2.y * t2.y);
    tt[2] = (float)(t1.z * t1.z + t2.z * t2.z); tt[3] = (float)(t1.x * t1.y + t2.x * t2.y);
    tt[4] = (float)(t1.x * t1.z + t2.x * t2.z); tt[5] = (float)(t1.y * t1.z + t2.y * t2.z);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (gid[k] >= 0) { key[k] = (unsigned)gid[k]; wf[k] = A.w[k]; }
    // indenter side: force f1 sig T tau on c, torque rho x (f1 T tau)
    d3 F = (f1 * sig) * Tt, tq = cross(rho, f1 * Tt);
    gr[0] += F.x; gr[1] += F.y; gr[2] += F.z; gr[3] += tq.x; gr[4] += tq.y; gr[5] += tq.z;
    add_sym(Dc, t1, f1 * sig * sig);
    add_sym(Dc, t2, f1 * sig * sig);
    add_sym(Dt, cross(rho, t1), f1);
    add_sym(Dt, cross(rho, t2), f1);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      float sc[9];
      const float fw = f1f * wf[k], sw = fw * wf[k];  // 0 for an absent corner (wf = 0)
#pragma unroll
      for (int c = 0; c < 3; ++c) sc[c] = fw * Ttf[c];
#pragma unroll
      for (int m = 0; m < 6; ++m) sc[3 + m] = sw * tt[m];
      seg_red9(d, e, key[k], sc);
    }
  }
  double vals[20];
  vals[0] = 0;
  vals[1] = Ef;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    vals[2 + k] = gr[k];
    vals[8 + k] = Dc[k];
    vals[14 + k] = Dt[k];
  }
  block_sums_contact(vals, d.acc, d.Es, e, smr);
}

// ---- staged contact passes (default when the env's surface fits in shared memory) ----
// One CTA per (env, chunk): the env's gel-surface displacements (float4 per surface
// vertex) and the rotated indenter vertices R Y (fp64) are staged in shared memory once,
// so every candidate reads its corners from shared memory instead of three scattered
// 32-byte sectors per gel corner.  Pass 1 classifies (separating-axis certificate ->
// g_min; otherwise a block-local near list), pass 2 runs the exact fp64 distances on
// convergent warps, pass 3 the friction anchors.
struct Stage {
  float4* sv4;  // [nsv] staged per-surface-vertex vector (u or p)
  float4* sy;   // [niv] R Y (fp32: only motion bounds and GN terms use it)
};
__device__ __forceinline__ Stage stage_ptrs(const Dev& d, char* sh) {
  Stage S;
  S.sy = reinterpret_cast<float4*>(sh);
  S.sv4 = reinterpret_cast<float4*>(sh + sizeof(float4) * d.niv);
  return S;
}
// staging loops issue kStageILP independent loads per thread before the shared stores
// (one load round trip per kStageILP x blockDim elements instead of one per blockDim)
constexpr int kStageILP = 4;
__device__ void stage_env(const Dev& d, const Stage& S, const float4* surf, int e, const double* R) {
  for (int i0 = threadIdx.x; i0 < d.nsv; i0 += kStageILP * blockDim.x) {
    float4 v[kStageILP];
#pragma unroll
    for (int k = 0; k < kStageILP; ++k) {
      const int i = i0 + k * blockDim.x;
      if (i < d.nsv) v[k] = surf[(size_t)i * d.Es + e];
    }
#pragma unroll
    for (int k = 0; k < kStageILP; ++k) {
      const int i = i0 + k * blockDim.x;
      if (i < d.nsv) S.sv4[i] = v[k];
    }
  }
  for (int j0 = threadIdx.x; j0 < d.niv; j0 += kStageILP * blockDim.x) {
    float4 yb[kStageILP];
#pragma unroll
    for (int k = 0; k < kStageILP; ++k) {
      const int j = j0 + k * blockDim.x;
      if (j < d.niv) yb[k] = __ldg(d.Y + j);
    }
#pragma unroll
    for (int k = 0; k < kStageILP; ++k) {
      const int j = j0 + k * blockDim.x;
      if (j < d.niv) {
        d3 y = mv(R, mk(yb[k].x, yb[k].y, yb[k].z));
        S.sy[j] = make_float4((float)y.x, (float)y.y, (float)y.z, 0.f);
      }
    }
  }
}

// staged classification.  Phase A reads each candidate's cached certificate h = g +
// odometer-at-certification: the pair's axis gap now is >= h - odo (the gap changes by at
// most the relative motion, which the odometer bounds along the path of evaluated
// points), so h - odo >= dhat keeps it far without touching its geometry (R15 cache).
// The rest (every pair after a new candidate list) is queued in shared memory and phase
// B runs the axis test on them densely with corners from shared memory: certificate ->
// cache refresh, otherwise the block-local near list of its kind, flushed with one global
// reservation per kind.  Work per CTA = chunks of kClassChunk candidates, so the number
// of dependent global round trips per CTA is a handful, not one per candidate batch.
constexpr int kClassChunk = 4096;  // candidates per chunk (queue offsets fit 16 bits)
constexpr int kClassA = kClassChunk / 256;  // phase-A candidates per thread
constexpr int kClassNL = 1024;     // block-local near-list capacity per kind and chunk
__device__ __forceinline__ void push_local(bool mine, int lane, int* cnt, unsigned short* list, int cap, int off,
                                           int* gcnt, uint2* glist, uint2 cw) {
  unsigned m = __ballot_sync(0xffffffffu, mine);
  if (!m) return;
  int slot0 = 0;
  if (lane == 0) slot0 = atomicAdd(cnt, __popc(m));
  slot0 = __shfl_sync(0xffffffffu, slot0, 0);
  const int slot = slot0 + __popc(m & ((1u << lane) - 1));
  if (!mine) return;
  if (slot < cap) list[slot] = (unsigned short)off;
  else glist[atomicAdd(gcnt, 1)] = cw;  // local list full: direct global append
}
// REMAP (tolerance mode): env_block's mapping and shorter chunks for a straggler's extra CTAs;
// the fixed mode's instantiation keeps the identity mapping and compile-time chunks (the
// runtime chunk length measured 171 -> 191 us per launch at C3)
template <bool BODY, bool REMAP>
__global__ void __launch_bounds__(256) k_contact_classify_staged(Dev d) {
  TAC_PDL_WAIT();
  // BODY: the test runs in the indenter's body frame (separation along an axis of any
  // orthonormal frame bounds the distance, R15): the env's gel surface is staged as
  // R^T (X + u - c) and the indenter corners are its static body-frame vertices Y, shared by
  // every env (L1/L2 resident) -- chosen when staging both sides would take more than 64 KB of
  // shared memory per CTA (C5: 113 KB, one CTA per SM).  Otherwise both sides are staged in the
  // gel frame (X + u, c + R Y; C3: 45 KB).  fp32 positions carry absolute errors
  // <= ~6e-9 m at the pad scale, so a pair is certified far only if its fp32 gap exceeds
  // dhat + kClassMargin and the cached gap is lowered by the same margin: conservative.
  constexpr float kClassMargin = 1e-7f;
  extern __shared__ __align__(16) char shc4[];
  __shared__ unsigned short q[kClassChunk];
  __shared__ unsigned short nl[3][kClassNL];
  __shared__ int qn, nn[3], nbase[3];
  __shared__ double Rs[9], cs[3];
  int e, bx, nbx;
  if constexpr (REMAP) {
    if (!env_block(d, 1, e, bx, nbx)) return;
  } else {
    e = blockIdx.y;
    bx = blockIdx.x;
    nbx = gridDim.x;
    if (e >= d.E || !(d.run[e] & 1)) return;
  }
  const int lb = d.lbuf[e];
  const int n = min(d.ncand[lb * d.E + e], d.kmax);
  // chunk length: kClassChunk, or less (>= 1024: every CTA stages the whole env) when the env
  // has more blocks than kClassChunk-chunks
  const int cl = REMAP ? min(kClassChunk, max(1024, ((n + nbx - 1) / nbx + 255) & ~255)) : kClassChunk;
  if (bx * cl >= n) return;  // no chunk: skip the staging
  const EnvS& s = d.es[e];
  float4* sx = reinterpret_cast<float4*>(shc4);                           // [nsv] gel surface
  float4* sy = reinterpret_cast<float4*>(shc4 + sizeof(float4) * d.nsv);  // [niv] c + R Y (gel frame only)
  if constexpr (BODY) {
    if (threadIdx.x < 9) Rs[threadIdx.x] = s.R[threadIdx.x];
    if (threadIdx.x < 3) cs[threadIdx.x] = s.c[threadIdx.x];
    __syncthreads();  // Rs, cs
    for (int i0 = threadIdx.x; i0 < d.nsv; i0 += kStageILP * blockDim.x) {
      float4 X[kStageILP], u[kStageILP];
#pragma unroll
      for (int k = 0; k < kStageILP; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i < d.nsv) { X[k] = __ldg(d.Xs + i); u[k] = d.usurf[(size_t)i * d.Es + e]; }
      }
#pragma unroll
      for (int k = 0; k < kStageILP; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i < d.nsv) {
          const d3 x = mk((double)X[k].x + (double)u[k].x - cs[0], (double)X[k].y + (double)u[k].y - cs[1],
                          (double)X[k].z + (double)u[k].z - cs[2]);
          sx[i] = make_float4((float)(Rs[0] * x.x + Rs[3] * x.y + Rs[6] * x.z),
                              (float)(Rs[1] * x.x + Rs[4] * x.y + Rs[7] * x.z),
                              (float)(Rs[2] * x.x + Rs[5] * x.y + Rs[8] * x.z), 0.f);
        }
      }
    }
  } else {
    if (threadIdx.x < 9) Rs[threadIdx.x] = s.R[threadIdx.x];
    if (threadIdx.x < 3) cs[threadIdx.x] = s.c[threadIdx.x];
    for (int i0 = threadIdx.x; i0 < d.nsv; i0 += kStageILP * blockDim.x) {
      float4 X[kStageILP], u[kStageILP];
#pragma unroll
      for (int k = 0; k < kStageILP; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i < d.nsv) { X[k] = __ldg(d.Xs + i); u[k] = d.usurf[(size_t)i * d.Es + e]; }
      }
#pragma unroll
      for (int k = 0; k < kStageILP; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i < d.nsv) sx[i] = make_float4(X[k].x + u[k].x, X[k].y + u[k].y, X[k].z + u[k].z, 0.f);
      }
    }
    __syncthreads();  // Rs, cs
    for (int j0 = threadIdx.x; j0 < d.niv; j0 += kStageILP * blockDim.x) {
      float4 yb[kStageILP];
#pragma unroll
      for (int k = 0; k < kStageILP; ++k) {
        const int j = j0 + k * blockDim.x;
        if (j < d.niv) yb[k] = __ldg(d.Y + j);
      }
#pragma unroll
      for (int k = 0; k < kStageILP; ++k) {
        const int j = j0 + k * blockDim.x;
        if (j < d.niv) {
          d3 y = mv(Rs, mk(yb[k].x, yb[k].y, yb[k].z)) + ld3(cs);
          sy[j] = make_float4((float)y.x, (float)y.y, (float)y.z, 0.f);
        }
      }
    }
  }
  const bool cached = s.cache_ok;
  const double odo = s.odo, thr = d.dhat + odo;
  const float dh = (float)d.dhat + kClassMargin;
  float* hc = d.cgap + (size_t)e * d.kmax;
  const uint2* ccorn = d.ccorn + cand_off(d, lb, e);
  int* gcnt = d.nnear + 3 * e;
  uint2* glist = d.nearl + (size_t)e * 3 * d.kmax;
  const int lane = threadIdx.x & 31;
  bool any_far = false;
  for (int c0 = bx * cl; c0 < n; c0 += nbx * cl) {
    if (threadIdx.x < 3) nn[threadIdx.x] = 0;
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();  // (also orders the staging above before phase B)
    // phase A: all cache loads first, then the decisions and the warp-aggregated queue push
    float h[kClassA];
#pragma unroll
    for (int k = 0; k < kClassA; ++k) {
      const int i = c0 + k * 256 + threadIdx.x;
      h[k] = (cached && i < n && k * 256 + (int)threadIdx.x < cl) ? hc[i] : -INFINITY;
    }
#pragma unroll
    for (int k = 0; k < kClassA; ++k) {
      const int off = k * 256 + threadIdx.x;
      const bool in = off < cl && c0 + off < n;
      const bool hit = in && (double)h[k] >= thr;
      any_far |= hit;
      const bool need = in && !hit;
      unsigned m = __ballot_sync(0xffffffffu, need);
      int slot0 = 0;
      if (lane == 0 && m) slot0 = atomicAdd(&qn, __popc(m));
      slot0 = __shfl_sync(0xffffffffu, slot0, 0);
      if (need) q[slot0 + __popc(m & ((1u << lane) - 1))] = (unsigned short)off;
    }
    __syncthreads();
    const int nq = qn;
    // phase B: queued pairs, two per thread in flight
    for (int jb = threadIdx.x & ~31; jb < nq; jb += 2 * blockDim.x) {
      int off[2], kind[2];
      uint2 cc[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int jq = jb + t * blockDim.x + lane;
        off[t] = jq < nq ? q[jq] : -1;
        kind[t] = 0;
        if (off[t] >= 0) { cc[t] = ccorn[c0 + off[t]]; kind[t] = (int)(cc[t].y >> 30); }
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        bool near = false;
        if (off[t] >= 0) {
          const int i = c0 + off[t];
          const unsigned id[4] = {cc[t].x & 0xffffu, cc[t].x >> 16, cc[t].y & 0xffffu, (cc[t].y >> 16) & 0x3fffu};
          // corner k is on the indenter: kind 0 (gel point, indenter triangle) k >= 1,
          // kind 1 (indenter point, gel triangle) k == 0, kind 2 (gel edge, indenter edge) k >= 2
          const int kd = kind[t], na = kd == 2 ? 2 : 1;
          float zx[4], zy[4], zz[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool ind = kd == 0 ? k >= 1 : (kd == 1 ? k == 0 : k >= 2);
            const float4 p = ind ? (BODY ? __ldg(d.Y + id[k]) : sy[id[k]]) : sx[id[k]];
            zx[k] = p.x; zy[k] = p.y; zz[k] = p.z;
          }
          float best = -INFINITY;
          const float* zs[3] = {zx, zy, zz};
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            const float* z = zs[ax];
            float loA = INFINITY, hiA = -INFINITY, loB = INFINITY, hiB = -INFINITY;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (k < na) { loA = fminf(loA, z[k]); hiA = fmaxf(hiA, z[k]); }
              else { loB = fminf(loB, z[k]); hiB = fmaxf(hiB, z[k]); }
            }
            best = fmaxf(best, fmaxf(loA - hiB, loB - hiA));
          }
          double gcert = (double)best;
          if (!(best >= dh)) {
            // no axis certificate: the primitive-plane gap in fp64 on the same fp32 corners
            // (moving each corner by <= eps changes the separation along any fixed normal by
            // <= 2 eps, so the margin keeps it conservative for the exact positions)
            d3 zd[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) zd[k] = mk(zx[k], zy[k], zz[k]);
            gcert = fmax(gcert, plane_gap(zd, na));
          }
          if (gcert >= (double)dh) {
            any_far = true;
            hc[i] = __double2float_rd((gcert - (double)kClassMargin) + odo);
          } else {
            near = true;
            if (!cached) hc[i] = -INFINITY;  // slot of a fresh list: never valid until re-certified
          }
        }
#pragma unroll
        for (int kk = 0; kk < 3; ++kk)  // per-kind near lists (convergent near-pair passes)
          push_local(near && kind[t] == kk, lane, &nn[kk], nl[kk], kClassNL, off[t], gcnt + kk,
                     glist + (size_t)kk * d.kmax, cc[t]);
      }
    }
    __syncthreads();
    if (threadIdx.x < 3) nbase[threadIdx.x] = atomicAdd(gcnt + threadIdx.x, min(nn[threadIdx.x], kClassNL));
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 3; ++kk) {
      const int m = min(nn[kk], kClassNL);
      for (int t = threadIdx.x; t < m; t += blockDim.x) glist[(size_t)kk * d.kmax + nbase[kk] + t] = ccorn[c0 + nl[kk][t]];
    }
    __syncthreads();  // q / nl / counters reuse
  }
  // far pairs share the bound (1 - s) dhat / L_rel (R15): only their existence is recorded
  if (__any_sync(0xffffffffu, any_far) && lane == 0) atomic_min_pos(d.accu + (size_t)U_GFAR * d.Es + e, (float)d.dhat);
}

// curvature + near-pair step bounds from the cached geometry, p staged in shared memory
__global__ void __launch_bounds__(256) k_contact_curv_staged(Dev d, double h2) {
  TAC_PDL_WAIT();
  extern __shared__ __align__(16) char shc3[];
  int e, bx, nbx;
  if (!env_block(d, 2, e, bx, nbx)) return;
  const double kappa = h2 * d.edbl[e];  // h^2 kappa_phys of this env
  const EnvS& s = d.es[e];
  __shared__ double R[9], pr[6];
  __shared__ double sm[8];
  if (threadIdx.x < 9) R[threadIdx.x] = s.R[threadIdx.x];
  if (threadIdx.x < 6) pr[threadIdx.x] = s.pr[threadIdx.x];
  __syncthreads();
  Stage S = stage_ptrs(d, shc3);
  stage_env(d, S, d.psurf, e, R);
  __syncthreads();
  d3 pc = mk(pr[0], pr[1], pr[2]), pth = mk(pr[3], pr[4], pr[5]);
  double extra = nrm(pth) * d.dhat * 0.25;
  // motion per unit alpha of corner id (indenter vertex or surface-local gel id)
  auto motion = [&](bool ind, unsigned id) -> d3 {
    if (ind) {
      const float4 y = S.sy[id];
      return pc + cross(pth, mk(y.x, y.y, y.z));
    }
    float4 p = S.sv4[id];
    return mk(p.x, p.y, p.z);
  };
  double q = 0, amin = INFINITY;
  const int n0 = d.nnear[3 * e], n1 = d.nnear[3 * e + 1], n = n0 + n1 + d.nnear[3 * e + 2];
  for (int j = bx * blockDim.x + threadIdx.x; j < n; j += nbx * blockDim.x) {
    const int kk = j < n0 ? 0 : (j < n0 + n1 ? 1 : 2);
    // near-ordered geometry and corners (written by k_contact_near at this position)
    const size_t slot = (size_t)e * d.kmax + j;
    const uint2 cc = d.ncorn[slot];
    const unsigned id[4] = {cc.x & 0xffffu, cc.x >> 16, cc.y & 0xffffu, (cc.y >> 16) & 0x3fffu};
    const int na = kk == 2 ? 2 : 1;
    const float4* geo = d.cgeo + 2 * slot;
    float4 g0 = geo[0], g1 = geo[1];
    double dist = g0.x;
    if (!(dist > 0)) continue;
    d3 nn = mk(g0.y, g0.z, g0.w);
    double w[4] = {g1.x, g1.y, g1.z, g1.w};
    d3 dz[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) dz[k] = motion(kk == 0 ? k >= 1 : (kk == 1 ? k == 0 : k >= 2), id[k]);
    if (dist < d.dhat) {
      d3 dr = mk(0, 0, 0);
#pragma unroll
      for (int k = 0; k < 4; ++k) dr = dr + w[k] * dz[k];
      double dn = dot(nn, dr);
      double lg = log(dist / d.dhat), dm = dist - d.dhat, inv = 1.0 / dist;
      q += kappa * (-2 * lg - 4 * dm * inv + dm * dm * inv * inv) * dn * dn;
    }
    double la = -INFINITY, lb = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < na) la = fmax(la, -dot(nn, dz[k]));
      else lb = fmax(lb, dot(nn, dz[k]));
    }
    double l = la + lb + extra;
    if (l > 0) amin = fmin(amin, (1 - d.ccd_s) * dist / l);
  }
  const int na = min(d.nanc[e], d.amax);
  for (int i = bx * blockDim.x + threadIdx.x; i < na; i += nbx * blockDim.x) {
    const Anchor& A = d.anc[(size_t)e * d.amax + i];
    const unsigned sid[3] = {A.sid01 & 0xffffu, A.sid01 >> 16, A.sid2};
    // indenter side folded: sig p_c + p_theta x (R Y_w)
    d3 dD = (double)A.sig * pc + cross(pth, mv(R, mk(A.yw[0], A.yw[1], A.yw[2])));
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (A.gid[k] >= 0) {
        const float4 pv = S.sv4[sid[k]];
        dD = dD + (double)A.w[k] * mk(pv.x, pv.y, pv.z);
      }
    d3 t1 = mk(A.t1[0], A.t1[1], A.t1[2]), t2 = mk(A.t2[0], A.t2[1], A.t2[2]);
    double ta = dot(t1, dD), tb = dot(t2, dD);
    q += (double)d.anc_f1[(size_t)e * d.amax + i] * (ta * ta + tb * tb);
  }
  // block reductions: sum q, min amin
  q = warp_sum(q);
  amin = warp_min(amin);
  __shared__ double smin[8];
  if ((threadIdx.x & 31) == 0) { sm[threadIdx.x >> 5] = q; smin[threadIdx.x >> 5] = amin; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0, m = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t += sm[w]; m = fmin(m, smin[w]); }
    if (t != 0.0) atomicAdd(d.acc + (size_t)A_PHP * d.Es + e, t);
    if (m < INFINITY) atomic_min_pos(d.accu + (size_t)U_ACCD * d.Es + e, (float)m);
  }
}

// curvature + near-pair step bounds from the cached geometry, corners gathered directly: the
// gel corners' p from the compact per-env surface copy (written by k_dir_apply just before,
// L2-resident), the indenter corners' R Y from the static body-frame vertices -- only the
// corners the env's near pairs and anchors touch, instead of staging its whole surface and
// indenter per CTA
__global__ void __launch_bounds__(128) k_contact_curv_direct(Dev d, double h2) {
  TAC_PDL_WAIT();
  int e, bx, nbx;
  if (!env_block(d, 2, e, bx, nbx)) return;
  const double kappa = h2 * d.edbl[e];  // h^2 kappa_phys of this env
  const EnvS& s = d.es[e];
  __shared__ double R[9], pr[6];
  __shared__ double sm[8];
  if (threadIdx.x < 9) R[threadIdx.x] = s.R[threadIdx.x];
  if (threadIdx.x < 6) pr[threadIdx.x] = s.pr[threadIdx.x];
  __syncthreads();
  d3 pc = mk(pr[0], pr[1], pr[2]), pth = mk(pr[3], pr[4], pr[5]);
  double extra = nrm(pth) * d.dhat * 0.25;
  // motion per unit alpha of corner id (indenter vertex or surface-local gel id)
  auto motion = [&](bool ind, unsigned id) -> d3 {
    if (ind) {  // fp32 R Y exactly as the staged pass rounds it
      const float4 yb = __ldg(d.Y + id);
      const d3 y = mv(R, mk(yb.x, yb.y, yb.z));
      return pc + cross(pth, mk((float)y.x, (float)y.y, (float)y.z));
    }
    const float4 p = d.psurf[(size_t)id * d.Es + e];
    return mk(p.x, p.y, p.z);
  };
  double q = 0, amin = INFINITY;
  const int n0 = d.nnear[3 * e], n1 = d.nnear[3 * e + 1], n = n0 + n1 + d.nnear[3 * e + 2];
  const int jstep = nbx * blockDim.x;
  uint2 cc_next = make_uint2(0u, 0u);
  if (bx * blockDim.x + threadIdx.x < n) cc_next = d.ncorn[(size_t)e * d.kmax + bx * blockDim.x + threadIdx.x];
  for (int j = bx * blockDim.x + threadIdx.x; j < n; j += jstep) {
    const int kk = j < n0 ? 0 : (j < n0 + n1 ? 1 : 2);
    // near-ordered geometry and corners (written by k_contact_near at this position); the next
    // round's corner word is loaded ahead
    const size_t slot = (size_t)e * d.kmax + j;
    const uint2 cc = cc_next;
    if (j + jstep < n) cc_next = d.ncorn[slot + jstep];
    const unsigned id[4] = {cc.x & 0xffffu, cc.x >> 16, cc.y & 0xffffu, (cc.y >> 16) & 0x3fffu};
    const int na = kk == 2 ? 2 : 1;
    const float4* geo = d.cgeo + 2 * slot;
    float4 g0 = geo[0], g1 = geo[1];
    double dist = g0.x;
    if (!(dist > 0)) continue;
    d3 nn = mk(g0.y, g0.z, g0.w);
    double w[4] = {g1.x, g1.y, g1.z, g1.w};
    d3 dz[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) dz[k] = motion(kk == 0 ? k >= 1 : (kk == 1 ? k == 0 : k >= 2), id[k]);
    if (dist < d.dhat) {
      d3 dr = mk(0, 0, 0);
#pragma unroll
      for (int k = 0; k < 4; ++k) dr = dr + w[k] * dz[k];
      double dn = dot(nn, dr);
      // b'' for the curvature estimate only (alpha_bar of P:461, then Armijo): fp32 log / rcp
      const float rf = (float)(dist / d.dhat), lgf = __logf(rf), invf = __frcp_rn(rf);
      const double dmr = (double)rf - 1.0;  // (d - dhat) / dhat
      const double ddb = (-2.0 * lgf - 4.0 * dmr * invf + dmr * dmr * invf * invf);
      q += kappa * ddb * dn * dn;
    }
    double la = -INFINITY, lb = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < na) la = fmax(la, -dot(nn, dz[k]));
      else lb = fmax(lb, dot(nn, dz[k]));
    }
    double l = la + lb + extra;
    if (l > 0) amin = fmin(amin, (1 - d.ccd_s) * dist / l);
  }
  const int na = min(d.nanc[e], d.amax);
  // (loading the next round's corner ids ahead here measured 116 -> 112 us per launch but the
  // step no faster: 94 instead of 80 registers)
  for (int i = bx * blockDim.x + threadIdx.x; i < na; i += jstep) {
    const Anchor& A = d.anc[(size_t)e * d.amax + i];
    const unsigned sid[3] = {A.sid01 & 0xffffu, A.sid01 >> 16, A.sid2};
    // indenter side folded: sig p_c + p_theta x (R Y_w)
    d3 dD = (double)A.sig * pc + cross(pth, mv(R, mk(A.yw[0], A.yw[1], A.yw[2])));
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (A.gid[k] >= 0) {
        const float4 pv = d.psurf[(size_t)sid[k] * d.Es + e];
        dD = dD + (double)A.w[k] * mk(pv.x, pv.y, pv.z);
      }
    d3 t1 = mk(A.t1[0], A.t1[1], A.t1[2]), t2 = mk(A.t2[0], A.t2[1], A.t2[2]);
    double ta = dot(t1, dD), tb = dot(t2, dD);
    q += (double)d.anc_f1[(size_t)e * d.amax + i] * (ta * ta + tb * tb);
  }
  // block reductions: sum q, min amin
  q = warp_sum(q);
  amin = warp_min(amin);
  __shared__ double smin[8];
  if ((threadIdx.x & 31) == 0) { sm[threadIdx.x >> 5] = q; smin[threadIdx.x >> 5] = amin; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0, m = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t += sm[w]; m = fmin(m, smin[w]); }
    if (t != 0.0) atomicAdd(d.acc + (size_t)A_PHP * d.Es + e, t);
    if (m < INFINITY) atomic_min_pos(d.accu + (size_t)U_ACCD * d.Es + e, (float)m);
  }
}

// ------------------------------------------------------------------ a8: Armijo accept (per env)
// E_k = inertia + elastic + barrier + friction + pose spring; accept if
// E <= E_prev + c1 alpha g^T p + eps_E |E_prev| (R14); otherwise halve alpha from x_k,
// after max_halvings go back to x_k and restart along -P g.
__device__ void sym6_to_9(const double* a, double* M) {
  M[0] = a[0]; M[4] = a[1]; M[8] = a[2];
  M[1] = M[3] = a[3]; M[2] = M[6] = a[4]; M[5] = M[7] = a[5];
}
__device__ void apply_pose(EnvS& s, double a) {  // (c, R) = (c_p + a p_c, exp([a p_theta]) R_p)
  for (int i = 0; i < 3; ++i) s.c[i] = s.cp[i] + a * s.pr[i];
  double Q[9];
  rodrigues(a * mk(s.pr[3], s.pr[4], s.pr[5]), Q);
  mm3(Q, s.Rp, s.R);
}

__global__ void k_accept(Dev d, double h) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  EnvS& s = d.es[e];
  double* A = d.acc;
  const size_t Es = d.Es;
  // every load of the common path before the first store (see k_dir_scalar)
  const int rb = d.run[e];
  double acc[28];
  for (int k = 0; k < 28; ++k) acc[k] = A[k * Es + e];
  double c[3], cs[3], R[9], Rs[9], lam[6];
  for (int k = 0; k < 3; ++k) { c[k] = s.c[k]; cs[k] = s.cs[k]; }
  for (int k = 0; k < 9; ++k) { R[k] = s.R[k]; Rs[k] = s.Rs[k]; }
  for (int k = 0; k < 6; ++k) lam[k] = s.lam[k];
  const int ncand_over = s.ncand_over, iter = s.iter, reeval = s.reeval;
  const double sE = s.E, salpha = s.alpha, sgp = s.gp_prev, sodo = s.odo;
  if (!(rb & 1)) return;
  double h2 = h * h;
  d3 dc = ld3(c) - ld3(cs);
  double RRs[9];
  mmT(R, Rs, RRs);
  d3 phi = so3_log(RRs);
  double wt = spring_w(nrm(dc), d.k_t, d.f_max), wr = spring_w(nrm(phi), d.k_r, d.t_max);
  double Eb = acc[A_EB];
  double Ep = h2 * (spring_e(nrm(dc), d.k_t, d.f_max) + spring_e(nrm(phi), d.k_r, d.t_max));
  const d3 lt = ld3(lam), lr = ld3(lam + 3);
  if (d.pose_al) Ep += h2 * (dot(lt, dc) + dot(lr, phi));  // multiplier term (R29)
  double E = acc[A_EIN] + acc[A_EEL] + Eb + acc[A_EF] + Ep;
  double gr[6], Dc6[6], Dt6[6];
  for (int k = 0; k < 6; ++k) gr[k] = acc[A_GR + k];
  for (int k = 0; k < 6; ++k) { Dc6[k] = acc[A_DR + k]; Dt6[k] = acc[A_DR + 6 + k]; }
  s.Ep[0] = acc[A_EIN]; s.Ep[1] = acc[A_EEL]; s.Ep[2] = Eb; s.Ep[3] = acc[A_EF];
  s.Ep[4] = Ep;
  for (int k = 0; k < 28; ++k) A[k * Es + e] = 0.0;
  if (ncand_over) {  // candidate or anchor capacity exceeded: pairs were dropped, the barrier
    // and the step bound no longer see them -- the step fails and rolls back (flag 32)
    s.flags |= kFlagOverflow;
    s.mode = kDone;
    s.back = 0;
    d.run[e] = 0;
    d.dalpha[e] = 0.f;
    return;
  }
  gr[0] += h2 * wt * dc.x; gr[1] += h2 * wt * dc.y; gr[2] += h2 * wt * dc.z;
  gr[3] += h2 * wr * phi.x; gr[4] += h2 * wr * phi.y; gr[5] += h2 * wr * phi.z;
  if (d.pose_al) {  // h^2 lam_t and h^2 J_l(phi)^-T lam_r (R29)
    const d3 gl = so3_jl_inv_T(phi, lr);
    gr[0] += h2 * lt.x; gr[1] += h2 * lt.y; gr[2] += h2 * lt.z;
    gr[3] += h2 * gl.x; gr[4] += h2 * gl.y; gr[5] += h2 * gl.z;
  }
  for (int k = 0; k < 3; ++k) { Dc6[k] += h2 * wt; Dt6[k] += h2 * wr; }
  s.iter = iter + 1;
  d.dalpha[e] = 0.f;
  bool first = (iter + 1 == 1);
  if ((first || reeval) && !isfinite(E)) {  // infeasible / NaN at the step start or at x_k: roll back
    s.flags |= isfinite(Eb) ? kFlagNaN : kFlagInfeas;
    s.mode = kDone;
    d.run[e] = 0;
    return;
  }
  bool ok = first || reeval || (isfinite(E) && E <= sE + d.c1 * salpha * sgp + d.eps_E * fabs(sE));
  s.cache_ok = 1;  // this evaluation classified every candidate of the current list
  if (ok) {
    s.odo_base = sodo;
    s.E = E;
    s.wt_acc = wt;
    s.wr_acc = wr;
    for (int k = 0; k < 6; ++k) s.gr[k] = gr[k];
    sym6_to_9(Dc6, s.Dc);
    sym6_to_9(Dt6, s.Dth);
    s.halv = 0;
    s.reeval = 0;
    s.accepted = 1;
    s.back = 0;
    d.run[e] = 2;
    return;
  }
  s.accepted = 0;
  s.back = -s.alpha;  // the rejected trial is x_k + alpha p
  d.accu[U_GFAR * Es + e] = 0x7f800000u;  // the next evaluation re-classifies
  s.halv += 1;
  s.odo_base = s.odo + s.alpha * s.Lc;  // the odometer path returns to x_k
  if (s.halv <= d.max_halv) {
    double an = 0.5 * s.alpha;
    s.odo = s.odo_base + an * s.Lc;
    s.S += (s.alpha - an) * s.Lc;  // candidate-list odometer: the path back from the trial (R16)
    s.S2 += (s.alpha - an) * s.Lc;  // (and the pending list's)
    d.dalpha[e] = (float)(an - s.alpha);
    s.alpha = an;
    apply_pose(s, an);
  } else {
    d.dalpha[e] = (float)(-s.alpha);
    s.S += s.alpha * s.Lc;
    s.S2 += s.alpha * s.Lc;
    s.alpha = 0;
    s.odo = s.odo_base;
    for (int i = 0; i < 3; ++i) s.c[i] = s.cp[i];
    for (int i = 0; i < 9; ++i) s.R[i] = s.Rp[i];
    s.restart = 1;
    s.reeval = 1;
    s.halv = 0;
  }
  d.run[e] = 1;
}

// ------------------------------------------------------------------ a6: direction
// P = 3x3 block inverse (default) or scalar Jacobi diag(H)^-1 (R9)

// P applied to two vectors (P g and P y share the block's inverse).  Surface vertices:
// P = (D + Dcon)^-1 formed in fp64 (R24: the contact block may exceed the elastic one by
// ~1e8); scalar Jacobi likewise from the fp64 diagonal.  Other vertices: fp32.
__device__ __forceinline__ float rcp_(float x) { return 1.f / x; }
__device__ __forceinline__ double rcp_(double x) { return __drcp_rn(x); }
template <typename T>
__device__ __forceinline__ void precond2(T a, T b, T c, T xy, T xz, T yz, int scalar, const float* x1, const float* x2,
                                         float* y1, float* y2) {
  if (scalar) {
    const T ia = rcp_(a), ib = rcp_(b), ic = rcp_(c);
    y1[0] = (float)(x1[0] * ia); y1[1] = (float)(x1[1] * ib); y1[2] = (float)(x1[2] * ic);
    y2[0] = (float)(x2[0] * ia); y2[1] = (float)(x2[1] * ib); y2[2] = (float)(x2[2] * ic);
    return;
  }
  const T c00 = b * c - yz * yz, c01 = xz * yz - xy * c, c02 = xy * yz - b * xz;
  const T c11 = a * c - xz * xz, c12 = xy * xz - a * yz, c22 = a * b - xy * xy;
  const T inv = rcp_(a * c00 + xy * c01 + xz * c02);
  y1[0] = (float)(inv * (c00 * x1[0] + c01 * x1[1] + c02 * x1[2]));
  y1[1] = (float)(inv * (c01 * x1[0] + c11 * x1[1] + c12 * x1[2]));
  y1[2] = (float)(inv * (c02 * x1[0] + c12 * x1[1] + c22 * x1[2]));
  y2[0] = (float)(inv * (c00 * x2[0] + c01 * x2[1] + c02 * x2[2]));
  y2[1] = (float)(inv * (c01 * x2[0] + c11 * x2[1] + c12 * x2[2]));
  y2[2] = (float)(inv * (c02 * x2[0] + c12 * x2[1] + c22 * x2[2]));
}

// Direction reduction: the dots g^T P y, y^T p, y^T P y, p^T g, g^T P g, g^T g, p^T p and
// max |P g| per env, and P g stored for k_dir_apply.  SURF = false: the vertices off the gel
// surface (and fixed-free surface vertices are skipped), fp32 block inverse, two vertices in
// flight; SURF = true: the free surface vertices (the list sv), whose P = (D + Dcon)^-1 is formed
// in fp64 (R24) -- on a side stream beside the first, so the fp64 inverse's registers no longer
// throttle the bulk of the vertices (one kernel with both: 80 registers, one vertex in flight)
template <bool SURF, bool TOL>
__global__ void __launch_bounds__(256) k_dir_reduce(Dev d) {
  TAC_PDL_WAIT();
  constexpr int NB = SURF ? 1 : 2;
  int e, by, nby;
  if (!env_lanes<TOL>(d, ((SURF ? d.nsv : d.nv) + 7) / 8, blockIdx.x, blockIdx.y, gridDim.y, e, by, nby)) return;
  bool act = e < d.E && (d.run[e] & 3);  // speculative: k_accept may run concurrently (see launch_eval)
  if (!__any_sync(0xffffffffu, act)) return;
  double gPy = 0, yp = 0, yPy = 0, pg = 0, gPg = 0, gg = 0, pp = 0;
  float pgmax = 0.f;
  const int stride = nby * 8;
  const int n = SURF ? d.nsv : d.nv;
  for (int i0 = by * 8 + threadIdx.y; i0 < n; i0 += NB * stride) {  // NB vertices in flight
    float g[NB][3], gq[NB][3], p[NB][3], D[NB][6];
    int vv[NB];
    bool ok[NB];
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int i = i0 + t * stride;
      ok[t] = false;
      if (!act || i >= n) continue;
      const int v = SURF ? d.sv[i] : i;
      const unsigned char fl = d.vflag[v];
      ok[t] = !(fl & 1) && (SURF || !(fl & 2));
      vv[t] = v;
      if (!ok[t]) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        g[t][c] = d.g[vidx(d, c, v, e)];
        gq[t][c] = d.gp[vidx(d, c, v, e)];
        p[t][c] = d.p[vidx(d, c, v, e)];
      }
#pragma unroll
      for (int c = 0; c < 6; ++c) D[t][c] = d.D[vidxD(d, c, v, e)];
    }
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      if (!ok[t]) continue;
      const int v = vv[t];
      float y[3], Pg[3], Py[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) y[c] = g[t][c] - gq[t][c];
      if constexpr (SURF) {
        const int sl = i0 + t * stride;  // surface-local id
        const float* A = D[t];
        float C[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) C[c] = d.Dcon[vidxS(d, c, sl, e)];
        precond2<double>((double)A[0] + C[0], (double)A[1] + C[1], (double)A[2] + C[2], (double)A[3] + C[3],
                         (double)A[4] + C[4], (double)A[5] + C[5], d.precond, g[t], y, Pg, Py);
      } else {
        precond2<float>(D[t][0], D[t][1], D[t][2], D[t][3], D[t][4], D[t][5], d.precond, g[t], y, Pg, Py);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) d.Pg[vidx(d, c, v, e)] = Pg[c];  // for k_dir_apply (speculative, like the dots)
      const float* gv = g[t];
      const float* pv = p[t];
      gPy += gv[0] * Py[0] + gv[1] * Py[1] + gv[2] * Py[2];
      yp += y[0] * pv[0] + y[1] * pv[1] + y[2] * pv[2];
      yPy += y[0] * Py[0] + y[1] * Py[1] + y[2] * Py[2];
      pg += pv[0] * gv[0] + pv[1] * gv[1] + pv[2] * gv[2];
      gPg += gv[0] * Pg[0] + gv[1] * Pg[1] + gv[2] * Pg[2];
      gg += gv[0] * gv[0] + gv[1] * gv[1] + gv[2] * gv[2];
      pp += pv[0] * pv[0] + pv[1] * pv[1] + pv[2] * pv[2];
      pgmax = fmaxf(pgmax, sqrtf(Pg[0] * Pg[0] + Pg[1] * Pg[1] + Pg[2] * Pg[2]));
    }
  }
  // reduce over threadIdx.y in shared memory, one atomic per (block, env)
  __shared__ double sm[8][8][32];
  __shared__ float smx[8][32];
  double vals[7] = {gPy, yp, yPy, pg, gPg, gg, pp};
  for (int k = 0; k < 7; ++k) sm[k][threadIdx.y][threadIdx.x] = vals[k];
  smx[threadIdx.y][threadIdx.x] = pgmax;
  __syncthreads();
  if (threadIdx.y == 0 && act) {
    for (int k = 0; k < 7; ++k) {
      double s = 0;
      for (int j = 0; j < 8; ++j) s += sm[k][j][threadIdx.x];
      atomicAdd(d.acc + (size_t)(A_DOT + k) * d.Es + e, s);
    }
    float m = 0.f;
    for (int j = 0; j < 8; ++j) m = fmaxf(m, smx[j][threadIdx.x]);
    atomic_max_pos(d.accu + (size_t)U_PGMAX * d.Es + e, m);
  }
}

__device__ void rigid_P(const EnvS& s, int scalar, const double* x, double* y) {  // blockdiag(Dc, Dth)^-1 x
  for (int b = 0; b < 2; ++b) {
    const double* M = b == 0 ? s.Dc : s.Dth;
    const double* xx = x + 3 * b;
    double* yy = y + 3 * b;
    if (scalar) {
      for (int i = 0; i < 3; ++i) yy[i] = xx[i] / M[4 * i];
      continue;
    }
    double c00 = M[4] * M[8] - M[5] * M[7], c01 = M[5] * M[6] - M[3] * M[8], c02 = M[3] * M[7] - M[4] * M[6];
    double c11 = M[0] * M[8] - M[2] * M[6], c12 = M[2] * M[3] - M[0] * M[5], c22 = M[0] * M[4] - M[1] * M[3];
    double inv = 1.0 / (M[0] * c00 + M[1] * c01 + M[2] * c02);
    yy[0] = inv * (c00 * xx[0] + c01 * xx[1] + c02 * xx[2]);
    yy[1] = inv * (c01 * xx[0] + c11 * xx[1] + c12 * xx[2]);
    yy[2] = inv * (c02 * xx[0] + c12 * xx[1] + c22 * xx[2]);
  }
}

// per env: convergence on |P g|_disp (R17), Dai-Kou beta with restarts (R13),
// rigid part of the direction
__device__ __forceinline__ void rigid_P_m(const double* Dc, const double* Dth, int scalar, const double* x, double* y) {
  for (int b = 0; b < 2; ++b) {  // blockdiag(Dc, Dth)^-1 x (rigid_P on register copies)
    const double* M = b == 0 ? Dc : Dth;
    const double* xx = x + 3 * b;
    double* yy = y + 3 * b;
    if (scalar) {
      for (int i = 0; i < 3; ++i) yy[i] = xx[i] / M[4 * i];
      continue;
    }
    double c00 = M[4] * M[8] - M[5] * M[7], c01 = M[5] * M[6] - M[3] * M[8], c02 = M[3] * M[7] - M[4] * M[6];
    double c11 = M[0] * M[8] - M[2] * M[6], c12 = M[2] * M[3] - M[0] * M[5], c22 = M[0] * M[4] - M[1] * M[3];
    double inv = 1.0 / (M[0] * c00 + M[1] * c01 + M[2] * c02);
    yy[0] = inv * (c00 * xx[0] + c01 * xx[1] + c02 * xx[2]);
    yy[1] = inv * (c01 * xx[0] + c11 * xx[1] + c12 * xx[2]);
    yy[2] = inv * (c02 * xx[0] + c12 * xx[1] + c22 * xx[2]);
  }
}
// One thread per env: every load is issued before the first store (a store through d.acc /
// d.es could alias a later load, so the compiler would otherwise keep each load behind the
// stores before it -- a chain of dependent memory round trips in a latency-bound kernel).
__global__ void k_dir_scalar(Dev d) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  const size_t Es = d.Es;
  EnvS& s = d.es[e];
  const int rb = d.run[e];
  double dt[7];
  for (int k = 0; k < 7; ++k) dt[k] = d.acc[(A_DOT + k) * Es + e];
  const float pgmax = __uint_as_float(d.accu[U_PGMAX * Es + e]);
  double gr[6], grp[6], pr[6], Dc[9], Dth[9];
  for (int k = 0; k < 6; ++k) { gr[k] = s.gr[k]; grp[k] = s.grp[k]; pr[k] = s.pr[k]; }
  for (int k = 0; k < 9; ++k) { Dc[k] = s.Dc[k]; Dth[k] = s.Dth[k]; }
  const int restart = s.restart, iter = s.iter, best_it = s.best_it;
  const double best_pg = s.best_pg, gPg_prev = s.gPg_prev;
  for (int k = 0; k < 7; ++k) d.acc[(A_DOT + k) * Es + e] = 0.0;
  d.accu[U_PGMAX * Es + e] = 0u;
  if (!(rb & 2)) return;  // not accepted: the speculative sums of k_dir_reduce are dropped
  double Pg[6], y[6], Py[6];
  rigid_P_m(Dc, Dth, d.precond, gr, Pg);
  for (int k = 0; k < 6; ++k) y[k] = gr[k] - grp[k];
  rigid_P_m(Dc, Dth, d.precond, y, Py);
  for (int k = 0; k < 6; ++k) {
    dt[0] += gr[k] * Py[k];
    dt[1] += y[k] * pr[k];
    dt[2] += y[k] * Py[k];
    dt[3] += pr[k] * gr[k];
    dt[4] += gr[k] * Pg[k];
    dt[5] += gr[k] * gr[k];
    dt[6] += pr[k] * pr[k];
  }
  double pgd = fmax((double)pgmax, nrm(mk(Pg[0], Pg[1], Pg[2])) + d.rho_max * nrm(mk(Pg[3], Pg[4], Pg[5])));
  s.pg = pgd;
  if (d.fixed_iters == 0) {
    if (pgd <= d.tol_x) {
      s.mode = kDone; s.flags |= 1; d.run[e] = 0;
      return;
    }
    if (pgd < best_pg * (1 - 1e-3)) { s.best_pg = pgd; s.best_it = iter; }
    else if (d.stagnation > 0 && iter - best_it > d.stagnation) {
      s.mode = kDone; s.flags |= 64; d.run[e] = 0;
      return;
    }
  }
  double gPy = dt[0], yp = dt[1], yPy = dt[2], pg = dt[3], gPg = dt[4], gg = dt[5], pp = dt[6];
  bool rs = restart || iter == 1;
  double beta = 0;
  if (!rs) {
    if (fabs(yp) <= 1e-30 * sqrt(gg) * sqrt(pp)) rs = true;
    else if (d.beta_rule == 1) beta = fmax(0.0, gPy / gPg_prev);
    else if (d.beta_rule == 2) beta = gPg / gPg_prev;
    else {
      beta = gPy / yp - (yPy / yp) * (pg / yp);
      if (d.beta_rule == 3) beta = fmax(beta, 0.5 * pg / pp);  // DK+ truncation (R28)
    }
    if (!isfinite(beta)) rs = true;
  }
  if (rs) beta = 0;
  double gp = -gPg + beta * pg;
  if (gp >= 0) { beta = 0; gp = -gPg; }
  s.restart = 0;
  s.beta = beta;
  d.beta[e] = (float)beta;
  s.gp_prev = gp;
  s.gPg_prev = gPg;
  for (int k = 0; k < 6; ++k) {
    pr[k] = -Pg[k] + (beta != 0 ? beta * pr[k] : 0.0);
    s.pr[k] = pr[k];
    s.grp[k] = gr[k];
  }
  d.pcf[e] = make_float4((float)pr[0], (float)pr[1], (float)pr[2], 0.f);
}

// p = -P g + beta p_prev; g_prev = g; M = max |p_v|, L_rel = max_surface |p_v - p_c|, inertia p^T M p
template <bool TOL>
__global__ void __launch_bounds__(256) k_dir_apply(Dev d) {
  TAC_PDL_WAIT();
  int e, by, nby;
  if (!env_lanes<TOL>(d, (d.nv + 7) / 8, blockIdx.x, blockIdx.y, gridDim.y, e, by, nby)) return;
  bool act = e < d.E && (d.run[e] & 2);
  if (!__any_sync(0xffffffffu, act)) return;
  float beta = act ? d.beta[e] : 0.f;
  float4 pc = act ? d.pcf[e] : make_float4(0, 0, 0, 0);
  float M = 0.f, L = 0.f;
  double q = 0;
  const int stride = nby * 8;
  for (int v0 = by * 8 + threadIdx.y; v0 < d.nv; v0 += 2 * stride) {  // loads of two vertices first
    float g[2][3], Pgv[2][3], po[2][3], m[2];
    int si[2];
    bool ok[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int v = v0 + t * stride;
      ok[t] = false;
      if (!act || v >= d.nv) continue;
      const unsigned char fl = d.vflag[v];
      ok[t] = !(fl & 1);
      if (!ok[t]) continue;
      m[t] = d.mass[v] * d.emat[2 * d.Es + e];
      si[t] = (fl & 2) ? d.sidx[v] : -1;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        g[t][c] = d.g[vidx(d, c, v, e)];
        po[t][c] = beta != 0.f ? d.p[vidx(d, c, v, e)] : 0.f;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) Pgv[t][c] = d.Pg[vidx(d, c, v, e)];
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (!ok[t]) continue;
      const int v = v0 + t * stride;
      float p[3];
      const float* Pg = Pgv[t];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned i = vidx(d, c, v, e);
        p[c] = beta != 0.f ? -Pg[c] + beta * po[t][c] : -Pg[c];
        d.p[i] = p[c];
        d.gp[i] = g[t][c];
      }
      const float pn = sqrtf(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
      M = fmaxf(M, pn);
      if (si[t] >= 0) {
        const float a = p[0] - pc.x, b = p[1] - pc.y, c = p[2] - pc.z;
        L = fmaxf(L, sqrtf(a * a + b * b + c * c));
        d.psurf[(size_t)si[t] * d.Es + e] = make_float4(p[0], p[1], p[2], 0.f);
      }
      q += (double)m[t] * (double)(pn * pn);
    }
  }
  __shared__ double sq[8][32];
  __shared__ float sM[8][32], sL[8][32];
  sq[threadIdx.y][threadIdx.x] = q;
  sM[threadIdx.y][threadIdx.x] = M;
  sL[threadIdx.y][threadIdx.x] = L;
  __syncthreads();
  if (threadIdx.y == 0 && act) {
    double t = 0;
    float m = 0.f, l = 0.f;
    for (int j = 0; j < 8; ++j) { t += sq[j][threadIdx.x]; m = fmaxf(m, sM[j][threadIdx.x]); l = fmaxf(l, sL[j][threadIdx.x]); }
    atomicAdd(d.acc + (size_t)A_PHP * d.Es + e, t);
    atomic_max_pos(d.accu + (size_t)U_M * d.Es + e, m);
    atomic_max_pos(d.accu + (size_t)U_LREL * d.Es + e, l);
  }
}


// ------------------------------------------------------------------ a7/a8: step length (per env)
// alpha = min(alpha_upper = dhat / (2 |p|_disp), alpha_bar = -g^T p / p^T H p,
// alpha_ccd (R15)); rebuild the candidates first if S + alpha L_rel > m_r (R16)

// R16: the candidate list stays valid while the odometer S <= m_r.  A step that would pass
// m_r is capped at it; once S + alpha L_rel passes kRebuildAt m_r the env is listed and its
// candidates are rebuilt at the state it moves to -- by k_broadphase_list right after the
// next k_vert_pre, on a side stream concurrent with the element pass.  kRebuildAt keeps a
// later cap from cutting a step below half of alpha_upper.
constexpr double kRebuildAt = 0.75;
__device__ void alpha_env(const Dev& d, double h, int e);
// tolerance mode: the block that finishes last lists the envs that evaluate next (run bit 0)
// and their groups for the next evaluation's block mappings (env_block / group_block)
__device__ void build_active_lists(const Dev& d) {
  __shared__ int last;
  __syncthreads();
  __threadfence();
  if (threadIdx.x == 0) last = atomicAdd(d.adone, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  const int lane = threadIdx.x;
  int n = 0, ng = 0;
  for (int base = 0; base < d.E; base += 1024) {
    int f[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int en = base + 32 * j + lane;
      f[j] = en < d.E ? __ldcg(d.run + en) : 0;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const unsigned m = __ballot_sync(0xffffffffu, f[j] & 1);
      if (f[j] & 1) d.alist[n + __popc(m & ((1u << lane) - 1))] = base + 32 * j + lane;
      n += __popc(m);
      if (m && lane == 0) d.glist[ng] = (base >> 5) + j;
      ng += m != 0u;
    }
  }
  if (lane == 0) {
    d.anum[0] = n;
    d.anum[1] = ng;
    *d.adone = 0u;
    if (d.loop_on) {  // WHILE body: continue while an env evaluates next (= is active) and trips remain
      const int c = ++(*d.loop_ctr);
      cudaGraphSetConditional(d.loop_h, (n > 0 && c < d.loop_limit) ? 1u : 0u);
    }
  }
}
__global__ void k_alpha(Dev d, double h) {
  TAC_PDL_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < d.E) alpha_env(d, h, e);
  if (d.fixed_iters <= 0) build_active_lists(d);
}
__device__ void alpha_env(const Dev& d, double h, int e) {
  const size_t Es = d.Es;
  EnvS& s = d.es[e];
  // every load before the first store (see k_dir_scalar)
  const int rb = d.run[e];
  double pr[6], c[3], R[9];
  for (int k = 0; k < 6; ++k) pr[k] = s.pr[k];
  for (int k = 0; k < 3; ++k) c[k] = s.c[k];
  for (int k = 0; k < 9; ++k) R[k] = s.R[k];
  const double wt_acc = s.wt_acc, wr_acc = s.wr_acc, gp_prev = s.gp_prev, S = s.S, S2 = s.S2, odo_base = s.odo_base;
  const int pending = s.pending, iter = s.iter, reb_iter = s.reb_iter;
  const double Mg = __uint_as_float(d.accu[U_M * Es + e]);
  const double Lg = __uint_as_float(d.accu[U_LREL * Es + e]);
  const double php = d.acc[A_PHP * Es + e];
  double accd = (double)__uint_as_float(d.accu[U_ACCD * Es + e]);
  const double gfar = (double)__uint_as_float(d.accu[U_GFAR * Es + e]);
  if (!(rb & 2)) return;
  double h2 = h * h;
  d3 pc = mk(pr[0], pr[1], pr[2]), pth = mk(pr[3], pr[4], pr[5]);
  double M = fmax(Mg, nrm(pc) + d.rho_max * nrm(pth));
  double L = fmax(Lg, nrm(pc)) + d.rho_max * nrm(pth);
  // the pose spring's Gauss-Newton curvature at x_k, with its weights from k_accept
  double q = php + h2 * (wt_acc * dot(pc, pc) + wr_acc * dot(pth, pth));
  d.acc[A_PHP * Es + e] = 0.0;
  d.accu[U_M * Es + e] = 0u;
  d.accu[U_LREL * Es + e] = 0u;
  if (gfar < INFINITY && L > 0) accd = fmin(accd, (1 - d.ccd_s) * d.dhat / L);  // far pairs (R15)
  d.accu[U_ACCD * Es + e] = 0x7f800000u;
  d.accu[U_GFAR * Es + e] = 0x7f800000u;
  double aup = M > 0 ? d.dhat / (2 * M) : INFINITY;
  double abar = q > 0 ? -gp_prev / q : INFINITY;
  double a = fmin(aup, fmin(abar, accd));
  if (!isfinite(a)) a = 0;
  s.dbg[0] = q; s.dbg[1] = M; s.dbg[2] = L; s.dbg[3] = aup; s.dbg[4] = abar; s.dbg[5] = accd; s.dbg[6] = a;
  // the list that will evaluate this step's trial: the pending one if it is swapped in first
  const bool swap_next = pending && iter >= reb_iter + 1;
  const double Sl = swap_next ? S2 : S;
  if (L > 0 && Sl + a * L > d.bp_margin) a = fmax(0.0, (d.bp_margin - Sl) / L);  // validity cap (R16)
  // commit: x_k -> (c_p, R_p); trial pose (c, R) = (c_p + a p_c, exp([a p_theta]) R_p)
  if (!isfinite(a)) a = 0;
  double cn[3], Rn[9], Q[9];
  for (int i = 0; i < 3; ++i) { s.cp[i] = c[i]; cn[i] = c[i] + a * pr[i]; s.c[i] = cn[i]; }
  rodrigues(a * pth, Q);
  mm3(Q, R, Rn);
  for (int i = 0; i < 9; ++i) { s.Rp[i] = R[i]; s.R[i] = Rn[i]; }
  s.alpha = a;
  d.dalpha[e] = (float)a;
  const double Sn = S + a * L;
  s.S = Sn;
  s.odo = odo_base + a * L;  // trial point x_k + a p on the odometer path
  s.Lc = L;
  d.run[e] = 1;
  if (!pending && L > 0 && Sn > kRebuildAt * d.bp_margin) {
    // pipelined rebuild (R16): a new list built at the trial point this step reaches, during the
    // next evaluation on a side stream (off its critical path), swapped in by the vertex pre-pass
    // of the evaluation after; until then the active list stays valid (S <= m_r, capped above)
    s.pending = 1;
    s.reb_iter = iter;
    s.S2 = 0;
    for (int i = 0; i < 3; ++i) s.cb[i] = cn[i];
    for (int i = 0; i < 9; ++i) s.Rb[i] = Rn[i];
    s.rebuild += 1;
    d.ncand[(1 - d.lbuf[e]) * d.E + e] = 0;
    d.reb_list[atomicAdd(d.nreb, 1)] = e;  // compact list for k_broadphase_list
  } else {
    s.S2 = S2 + a * L;
  }
}

// ------------------------------------------------------------------ a9: finalize
__global__ void k_finalize_vert(Dev d, float inv_h) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * 32 + threadIdx.x;
  if (e >= d.E) return;
  bool failed = d.es[e].flags & kFlagFailed;
  // commit the last accepted iterate x_k: the last evaluated point moved back by a rejected
  // trial's alpha (never the pending, unevaluated trial of the dalpha buffer)
  float da = (float)d.es[e].back;
  for (int v = blockIdx.y * 8 + threadIdx.y; v < d.nv; v += gridDim.y * 8) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      unsigned i = vidx(d, c, v, e);
      float ut = d.ut[i];
      if (failed) {
        d.u[i] = ut;
        d.vt[i] = 0.f;
        continue;
      }
      float u = d.u[i];
      if (da != 0.f) u += da * d.p[i];
      d.u[i] = u;
      d.vt[i] = (u - ut) * inv_h;
      d.ut[i] = u;
    }
  }
}
__global__ void k_finalize_env(Dev d) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  EnvS& s = d.es[e];
  if (s.flags & kFlagFailed) {
    for (int i = 0; i < 3; ++i) s.c[i] = s.ct[i];
    for (int i = 0; i < 9; ++i) s.R[i] = s.Rt[i];
  } else if (s.back != 0) {  // the last evaluation rejected its trial: x_k's pose
    for (int i = 0; i < 3; ++i) s.ct[i] = s.c[i] = s.cp[i];
    for (int i = 0; i < 9; ++i) s.Rt[i] = s.R[i] = s.Rp[i];
  } else {
    for (int i = 0; i < 3; ++i) s.ct[i] = s.c[i];
    for (int i = 0; i < 9; ++i) s.Rt[i] = s.R[i];
  }
  if (s.mode == kActive) s.flags |= kFlagMaxIt;
  s.ncand_max = max(s.ncand_max, d.ncand[d.lbuf[e] * d.E + e]);
  s.nanc_last = d.nanc[e];
  s.mode = kDone;
  d.run[e] = 0;
  d.dalpha[e] = 0.f;
  d3 dc = ld3(s.c) - ld3(s.cs);
  double RRs[9];
  mmT(s.R, s.Rs, RRs);
  const d3 phi = so3_log(RRs);
  s.pose_res = nrm(dc) + d.rho_max * nrm(phi);
  if (d.pose_al && !(s.flags & kFlagFailed)) {  // R29: lam += psi'(r) r/|r| at the step's solution
    const double wt = spring_w(nrm(dc), d.k_t, d.f_max), wr = spring_w(nrm(phi), d.k_r, d.t_max);
    s.lam[0] += wt * dc.x; s.lam[1] += wt * dc.y; s.lam[2] += wt * dc.z;
    s.lam[3] += wr * phi.x; s.lam[4] += wr * phi.y; s.lam[5] += wr * phi.z;
  }
}

// ------------------------------------------------------------------ a10: markers
// u_m = sum_j w_mj u_j; out[e][m] = (u_m.t1, u_m.t2[, u_m.n])
__global__ void k_markers(Dev d, float* out, int ncomp, float4 t1, float4 t2, float4 nn) {
  TAC_PDL_WAIT();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.E * d.nm) return;
  int e = i / d.nm, m = i - e * d.nm;
  int4 id = __ldg(d.mk_idx + m);
  float4 w = __ldg(d.mk_w + m);
  int vv[4] = {id.x, id.y, id.z, id.w};
  float ww[4] = {w.x, w.y, w.z, w.w};
  float um[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) um[c] = fmaf(ww[k], d.ut[vidx(d, c, vv[k], e)], um[c]);
  float* o = out + (size_t)i * ncomp;
  o[0] = um[0] * t1.x + um[1] * t1.y + um[2] * t1.z;
  o[1] = um[0] * t2.x + um[1] * t2.y + um[2] * t2.z;
  if (ncomp == 3) o[2] = um[0] * nn.x + um[1] * nn.y + um[2] * nn.z;
}

// calibration loss term (Eq. 6): acc[e] += sum_m |u_m(theta_e) - u_ref[e][m]|^2 over
// the marker field computed exactly as k_markers does; one CTA per env (sole writer)
__global__ void __launch_bounds__(128) k_marker_sqerr(Dev d, const float* ref, double* acc, int ncomp, float4 t1,
                                                      float4 t2, float4 nn) {
  TAC_PDL_WAIT();
  const int e = blockIdx.x;
  __shared__ double sw[4];
  double se = 0;
  for (int m = threadIdx.x; m < d.nm; m += blockDim.x) {
    int4 id = __ldg(d.mk_idx + m);
    float4 w = __ldg(d.mk_w + m);
    int vv[4] = {id.x, id.y, id.z, id.w};
    float ww[4] = {w.x, w.y, w.z, w.w};
    float um[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) um[c] = fmaf(ww[k], d.ut[vidx(d, c, vv[k], e)], um[c]);
    float o[3];
    o[0] = um[0] * t1.x + um[1] * t1.y + um[2] * t1.z;
    o[1] = um[0] * t2.x + um[1] * t2.y + um[2] * t2.z;
    o[2] = um[0] * nn.x + um[1] * nn.y + um[2] * nn.z;
    const float* r = ref + ((size_t)e * d.nm + m) * ncomp;
    for (int c = 0; c < ncomp; ++c) {
      const double df = (double)o[c] - (double)r[c];
      se += df * df;
    }
  }
  se = warp_sum(se);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = se;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sw[w];
    acc[e] += t;
  }
}

__global__ void k_reset_env(Dev d, const unsigned char* mask, const float* poses) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E || !mask[e]) return;
  EnvS& s = d.es[e];
  const float* q = poses + 7 * e;
  for (int i = 0; i < 3; ++i) s.ct[i] = s.c[i] = q[i];
  quat_R(q, s.Rt);
  for (int i = 0; i < 9; ++i) s.R[i] = s.Rt[i];
  s.flags = 0;
  s.iter = 0;
  s.pg = 0;
  for (int i = 0; i < 6; ++i) s.lam[i] = 0.0;
}
__global__ void k_reset_vert(Dev d, const unsigned char* mask) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * 32 + threadIdx.x;
  if (e >= d.E || !mask[e]) return;
  for (int v = blockIdx.y * 8 + threadIdx.y; v < d.nv; v += gridDim.y * 8)
    for (int c = 0; c < 3; ++c) {
      unsigned i = vidx(d, c, v, e);
      d.u[i] = d.ut[i] = d.vt[i] = d.p[i] = d.gp[i] = 0.f;
    }
}
__global__ void k_status(Dev d, int* iters, float* pg, unsigned* flags) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  if (iters) iters[e] = d.es[e].iter;
  if (pg) pg[e] = (float)d.es[e].pg;
  if (flags) flags[e] = (unsigned)d.es[e].flags;
}
__global__ void k_stats(Dev d, int4* out) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  const EnvS& s = d.es[e];
  out[e] = make_int4(s.iter, s.ncand_max, s.nanc_last, s.rebuild);
}
__global__ void k_any_active(Dev d, int* out) {
  TAC_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  int a = (e < d.E && d.es[e].mode == kActive) ? 1 : 0;
  if (__any_sync(0xffffffffu, a) && (threadIdx.x & 31) == 0) atomicOr(out, 1);
}

// tolerance mode's device-side loop control (body of the CUDA-graph WHILE node, tac_step):
// continue while any env is still iterating and fewer than `limit` iterations have run
__global__ void __launch_bounds__(1024) k_loop_ctl(Dev d, cudaGraphConditionalHandle h, int* ctr, int limit) {
  TAC_PDL_WAIT();
  int a = 0;
  for (int e = threadIdx.x; e < d.E; e += blockDim.x) a |= d.es[e].mode == kActive;
  a = __syncthreads_or(a);
  if (threadIdx.x == 0) {
    const int c = ++(*ctr);
    cudaGraphSetConditional(h, (a && c < limit) ? 1u : 0u);
  }
}

struct Words8 { uint64_t w[8]; };
__global__ void k_write_words(uint64_t* dst, Words8 v, int n) {
  TAC_PDL_WAIT();
  if (threadIdx.x < n) dst[threadIdx.x] = v.w[threadIdx.x];
}

// ------------------------------------------------------------------ launchers
static int env_int(const char* k, int dflt) { return getenv(k) ? atoi(getenv(k)) : dflt; }  // A/B
static dim3 vgrid(const Dev& d, int n, int bps = 8) {
  int gx = d.Es / 32;
  // ~8 blocks of 256 threads per SM over the grid (grid-stride over the rest); interleaved
  // A/B on B200 vs 16/SM: C3 +1.5 %, C5 +2.6 % (4/SM and 6/SM were slower, 12/SM within 0.3 %)
  int gy = (148 * bps + gx - 1) / gx;
  gy = std::max(1, std::min(gy, (n + 7) / 8));
  return dim3(gx, gy);
}
static dim3 cellgrid(const Dev& d) {
  static const int bps = env_int("TAC_CELL_BPS", 8);
  return vgrid(d, d.ncells, bps);
}
static dim3 cgrid(const Dev& d) {
  // ~contact_bps blocks of 128 threads per SM over the grid (per simulator: TAC_CONTACT_BPS at
  // tac_create, default 8 -- one block per env at 1,024 envs; interleaved A/B on C3: 20,897 vs
  // 20,526 env-steps/s at 16; converged parity is tested at both settings)
  const int tot = 148 * d.contact_bps;
  int nb = std::max(1, std::min(64, tot / std::max(1, d.E)));
  return dim3(nb, d.E);
}
static int eblocks(const Dev& d) { return (d.E + 127) / 128; }
// per-env control kernels (long serial fp64 chains per thread): one warp per block spreads
// the envs over E / 32 SMs instead of E / 128
static int eblocks32(const Dev& d) { return (d.E + 31) / 32; }
static dim3 sgrid(const Dev& d) {  // staged contact kernels: chunks per env
  // every CTA stages its env once, so CTAs per env stay few: one at 1,024+ envs (measured
  // +1.2 % at C3 against two), up to 16 for small batches
  static const int cap = getenv("TAC_SGRID_CAP") ? atoi(getenv("TAC_SGRID_CAP")) : 16;  // A/B experiments
  int nb = std::max(1, std::min(cap, 1184 / std::max(1, d.E)));
  return dim3(nb, d.E);
}
// Every launch is a programmatic dependent launch: the next kernel's CTAs may be resident
// while this one drains, and each kernel starts with griddepcontrol.wait (TAC_PDL_WAIT),
// which blocks until its stream predecessor has completed and flushed.  Memsets and
// profiling events between kernels fall back to ordinary stream serialisation.
template <typename... KArgs, typename... Args>
static void pdl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
#define LAUNCHP(kid, s, kern, grid, block, smem, ...)      \
  do {                                                   \
    if (g_prof) prof_begin(kid, s);                      \
    pdl_launch(kern, dim3(grid), dim3(block), (size_t)(smem), s, ##__VA_ARGS__); \
    if (g_prof) prof_end(kid, s);                        \
    if (g_tl_on) tl_mark(kid, s);                        \
    ++g_launches;                                        \
  } while (0)

void launch_step_setup(const Dev& d, const float* poses, double h, unsigned long long step, cudaStream_t s) {
  LAUNCHP(KID_STEP_SETUP, s, k_step_setup, eblocks32(d), 32, 0, d, poses, step);
  LAUNCHP(KID_VERT_SETUP, s, k_vert_setup, vgrid(d, d.nv), dim3(32, 8), 0, d, (float)h);
}
void launch_vert_setup(const Dev& d, double h, cudaStream_t s) {
  LAUNCHP(KID_VERT_SETUP, s, k_vert_setup, vgrid(d, d.nv), dim3(32, 8), 0, d, (float)h);
}
void launch_broadphase(const Dev& d, bool masked, cudaStream_t s) {
  if (masked) {  // envs listed by k_alpha; off the critical path (R16 pipeline): a small grid
    static const int bps = env_int("TAC_REB_BPS", 16), chunk = env_int("TAC_REB_CHUNK", 32);  // A/B
    LAUNCHP(KID_BROADPHASE_LIST, s, k_broadphase_list, bps * 148, 128, 0, d, d.dhat + d.bp_margin, chunk);
    return;
  }
  int ntot = d.nsv + d.nse + d.nst;
  static const int tot = env_int("TAC_BP_BLOCKS", 4736);  // A/B
  int nb = std::max(1, std::min((ntot + 127) / 128, tot / std::max(1, d.E)));
  LAUNCHP(KID_BROADPHASE, s, k_broadphase, dim3(nb, d.E), 128, 0, d, d.dhat + d.bp_margin, nullptr, nullptr, 0);
}
void launch_intersect_check(const Dev& d, int* hit, cudaStream_t s) {
  LAUNCHP(KID_OTHER, s, k_intersect_check, dim3((d.nse + 127) / 128, d.E), 128, 0, d, hit);
}
void launch_anchors(const Dev& d, double h, cudaStream_t s) {
  // once per step over the whole candidate lists: 16 CTAs per env (or the contact grid's, if
  // more) -- one CTA per env, the contact passes' grid at 1,024 envs, measured 0.90 vs 0.75 ms
  // per step for the anchors and their sort (TAC_ANC_NB for A/B)
  static const int nb = env_int("TAC_ANC_NB", 16);
  LAUNCHP(KID_ANCHORS, s, k_anchors, dim3(std::max((int)cgrid(d).x, nb), d.E), 128, 0, d, h * h);
}
void launch_sort_anchors(const Dev& d, Anchor* out, cudaStream_t s) {
  int n = 1;
  while (n < d.amax) n <<= 1;
  LAUNCHP(KID_ANCHORS, s, k_sort_anchors, d.E, 1024, sizeof(unsigned long long) * n, d, out);
}
// The element pass and the contact chain of an evaluation (and of the curvature pass) are
// independent -- both start from the positions k_vert_pre reached and add into g, D and the
// energy accumulators with atomics -- so the contact chain (with the candidate rebuild it
// depends on) runs on the high-priority side stream concurrently with the element kernels,
// joined before k_accept / k_alpha.  With per-launch profiling on, everything stays on the
// caller's stream so each kernel's time is its own.
void launch_eval(const Dev& d, double h, cudaStream_t s) {
  if (d.fixed_iters > 0) LAUNCHP(KID_VERT_PRE, s, k_vert_pre<false>, vgrid(d, d.nv), dim3(32, 8), 0, d, (float)(h * h));
  else LAUNCHP(KID_VERT_PRE, s, k_vert_pre<true>, vgrid(d, d.nv), dim3(32, 8), 0, d, (float)(h * h));
  const bool fork = g_prof == nullptr;
  cudaStream_t cs = fork ? d.side : s, cs2 = fork ? d.side2 : s;
  if (fork) {
    cudaEventRecord(d.ev_fork, s);
    cudaStreamWaitEvent(cs, d.ev_fork, 0);
    cudaStreamWaitEvent(cs2, d.ev_fork, 0);
  }
  // friction needs only the anchors (fixed for the step) and the surface displacements
  LAUNCHP(KID_CONTACT_FRICTION, cs2, k_contact_friction, cgrid(d), 128, 0, d, d.eps_v * h);
  // R16: candidates of the envs k_alpha listed, rebuilt at the trial state k_vert_pre just
  // reached into their spare buffer, on a third stream beside the whole evaluation (joined before
  // k_alpha; swapped in by the next k_vert_pre) -- not ahead of the classification any more
  cudaStream_t rs = fork ? d.side3 : s;
  if (fork) cudaStreamWaitEvent(rs, d.ev_fork, 0);
  launch_broadphase(d, true, rs);
  if (fork) cudaEventRecord(d.ev_reb, rs);
  const size_t cls_both = sizeof(float4) * (size_t)(d.nsv + d.niv);  // [nsv] X + u, [niv] c + R Y
  const bool remap = d.fixed_iters <= 0;
  if (cls_both > 64 * 1024) {  // body frame: stage the gel side only
    if (remap) LAUNCHP(KID_CONTACT_CLASSIFY, cs, (k_contact_classify_staged<true, true>), sgrid(d), 256, sizeof(float4) * (size_t)d.nsv, d);
    else LAUNCHP(KID_CONTACT_CLASSIFY, cs, (k_contact_classify_staged<true, false>), sgrid(d), 256, sizeof(float4) * (size_t)d.nsv, d);
  } else {
    if (remap) LAUNCHP(KID_CONTACT_CLASSIFY, cs, (k_contact_classify_staged<false, true>), sgrid(d), 256, cls_both, d);
    else LAUNCHP(KID_CONTACT_CLASSIFY, cs, (k_contact_classify_staged<false, false>), sgrid(d), 256, cls_both, d);
  }
  const double kap = h * h;  // kernels scale by their env's kappa_phys
  // the three near-pair passes are independent (atomics into g / Dcon): edge-edge after the
  // classification on its stream, gel-ind point-triangle after the friction pass, ind-gel on a
  // fourth stream (one dependent launch less in a tolerance-mode tail iteration)
  static const bool four = getenv("TAC_NO_SIDE4") == nullptr;
  cudaStream_t cs4 = fork && four ? d.side4 : cs2;
  if (fork) {
    cudaEventRecord(d.ev_cls, cs);
    cudaStreamWaitEvent(cs2, d.ev_cls, 0);
    if (four) cudaStreamWaitEvent(cs4, d.ev_cls, 0);
  }
  if (d.ee_moll) LAUNCHP(KID_CONTACT_NEAR_EE, cs, (k_contact_near<2, true>), cgrid(d), 128, 0, d, kap);
  else LAUNCHP(KID_CONTACT_NEAR_EE, cs, k_contact_near<2>, cgrid(d), 128, 0, d, kap);
  LAUNCHP(KID_CONTACT_GRAD, cs2, k_contact_near<0>, cgrid(d), 128, 0, d, kap);
  LAUNCHP(KID_CONTACT_NEAR_IG, cs4, k_contact_near<1>, cgrid(d), 128, 0, d, kap);
  if (fork) {
    cudaEventRecord(d.ev_join, cs);
    cudaEventRecord(d.ev_join2, cs2);
    if (four) cudaEventRecord(d.ev_join4, cs4);
  }
  // (a round-scheduled shared-memory tiled variant measured slower on C3: 740 vs 520 us at
  // 66 % warp utilisation in the rounds and 2 CTAs/SM; the coalesced red.add scatter stays)
  if (d.ncells > 0) {
    dim3 g = cellgrid(d);
    if (d.rows) {
      const int gy = (d.nseg + kRowWarps - 1) / kRowWarps;  // one segment per warp
      if (d.fixed_iters > 0) LAUNCHP(KID_ELEM_GRAD, s, k_elem_grad_rows<false>, dim3(gy, g.x), dim3(32, kRowWarps), 0, d, (float)(h * h));
      else LAUNCHP(KID_ELEM_GRAD, s, k_elem_grad_rows<true>, dim3(gy, g.x), dim3(32, kRowWarps), 0, d, (float)(h * h));
    } else if (d.cells_all_aa) LAUNCHP(KID_ELEM_GRAD, s, k_elem_grad_cells<true>, dim3(g.y, g.x), dim3(32, 8), 0, d, (float)(h * h));
    else LAUNCHP(KID_ELEM_GRAD, s, k_elem_grad_cells<false>, dim3(g.y, g.x), dim3(32, 8), 0, d, (float)(h * h));
  }
  if (d.nrest > 0) {
    dim3 g = vgrid(d, d.nrest);
    LAUNCHP(KID_ELEM_GRAD, s, k_elem_grad, dim3(g.y, g.x), dim3(32, 8), 0, d, (float)(h * h));
  }
  if (fork) {
    cudaStreamWaitEvent(s, d.ev_join, 0);
    cudaStreamWaitEvent(s, d.ev_join2, 0);
    if (four) cudaStreamWaitEvent(s, d.ev_join4, 0);
    // the Armijo decision (one thread per env, a latency-bound fp64 chain) runs on the side
    // stream beside the direction reduction, which sums its dots speculatively for every env
    // under evaluation; k_dir_scalar (after both) keeps the accepted envs' sums only
    cudaEventRecord(d.ev_cls, s);
    cudaStreamWaitEvent(cs, d.ev_cls, 0);
    LAUNCHP(KID_ACCEPT, cs, k_accept, eblocks32(d), 32, 0, d, h);
    cudaEventRecord(d.ev_join, cs);
  } else {
    LAUNCHP(KID_ACCEPT, s, k_accept, eblocks32(d), 32, 0, d, h);
  }
}
void launch_direction(const Dev& d, cudaStream_t s, bool apply) {
  // the surface vertices' fp64-preconditioned part beside the bulk (joined before k_dir_scalar)
  const bool fork = g_prof == nullptr;
  cudaStream_t ss = fork ? d.side2 : s;
  if (fork) {
    cudaEventRecord(d.ev_fork, s);
    cudaStreamWaitEvent(ss, d.ev_fork, 0);
  }
  static const int sbps = env_int("TAC_DIRS_BPS", 2);  // A/B
  if (d.fixed_iters > 0) LAUNCHP(KID_DIR_REDUCE_SURF, ss, (k_dir_reduce<true, false>), vgrid(d, std::max(1, d.nsv), sbps), dim3(32, 8), 0, d);
  else LAUNCHP(KID_DIR_REDUCE_SURF, ss, (k_dir_reduce<true, true>), vgrid(d, std::max(1, d.nsv), sbps), dim3(32, 8), 0, d);
  if (fork) cudaEventRecord(d.ev_join2, ss);
  if (d.fixed_iters > 0) LAUNCHP(KID_DIR_REDUCE, s, (k_dir_reduce<false, false>), vgrid(d, d.nv), dim3(32, 8), 0, d);
  else LAUNCHP(KID_DIR_REDUCE, s, (k_dir_reduce<false, true>), vgrid(d, d.nv), dim3(32, 8), 0, d);
  if (fork) {
    cudaStreamWaitEvent(s, d.ev_join, 0);   // k_accept on the side stream
    cudaStreamWaitEvent(s, d.ev_join2, 0);  // the surface part
  }
  LAUNCHP(KID_DIR_SCALAR, s, k_dir_scalar, eblocks32(d), 32, 0, d);
  if (apply) {
    if (d.fixed_iters > 0) LAUNCHP(KID_DIR_APPLY, s, k_dir_apply<false>, vgrid(d, d.nv), dim3(32, 8), 0, d);
    else LAUNCHP(KID_DIR_APPLY, s, k_dir_apply<true>, vgrid(d, d.nv), dim3(32, 8), 0, d);
  }
}
void launch_curvature(const Dev& d, double h, cudaStream_t s) {
  const bool fork = g_prof == nullptr;  // contact curvature concurrent with the element curvature
  cudaStream_t cs = fork ? d.side : s;
  if (fork) {
    cudaEventRecord(d.ev_fork, s);
    cudaStreamWaitEvent(cs, d.ev_fork, 0);
  }
  static const bool staged = getenv("TAC_CURV_STAGED") != nullptr;  // A/B: the staged variant
  if (staged) LAUNCHP(KID_CONTACT_CURV, cs, k_contact_curv_staged, sgrid(d), 256, d.contact_smem, d, h * h);
  else LAUNCHP(KID_CONTACT_CURV, cs, k_contact_curv_direct, cgrid(d), 128, 0, d, h * h);
  if (fork) cudaEventRecord(d.ev_join, cs);
  if (d.nrest == 0) {  // every tet is in a Kuhn cell: register-blocked cells
    dim3 g = cellgrid(d);
    // (a row-marching curvature pass -- u and p of the shared face carried -- measured 125 vs
    // 114 us: this pass is FMA-bound and the carried rows cost spills)
    const bool tol = d.fixed_iters <= 0;
    if (d.cells_all_aa && tol) LAUNCHP(KID_ELEM_CURV, s, (k_elem_curv_cells<true, true>), dim3(g.y, g.x), dim3(32, 8), 0, d, (float)(h * h));
    else if (d.cells_all_aa) LAUNCHP(KID_ELEM_CURV, s, (k_elem_curv_cells<true, false>), dim3(g.y, g.x), dim3(32, 8), 0, d, (float)(h * h));
    else if (tol) LAUNCHP(KID_ELEM_CURV, s, (k_elem_curv_cells<false, true>), dim3(g.y, g.x), dim3(32, 8), 0, d, (float)(h * h));
    else LAUNCHP(KID_ELEM_CURV, s, (k_elem_curv_cells<false, false>), dim3(g.y, g.x), dim3(32, 8), 0, d, (float)(h * h));
  } else {
    LAUNCHP(KID_ELEM_CURV, s, k_elem_curv_tiled, dim3(d.Es / 32, d.ntiles), 256, kTiledCurvSmem, d, (float)(h * h));
  }
  if (fork) cudaStreamWaitEvent(s, d.ev_join, 0);
}
void launch_alpha(const Dev& d, double h, cudaStream_t s) {
  if (g_prof == nullptr) cudaStreamWaitEvent(s, d.ev_reb, 0);  // the pipelined rebuild has finished
  cudaMemsetAsync(d.nreb, 0, sizeof(int), s);
  LAUNCHP(KID_ALPHA, s, k_alpha, eblocks32(d), 32, 0, d, h);
}
void launch_finalize(const Dev& d, double h, cudaStream_t s) {
  LAUNCHP(KID_FIN_VERT, s, k_finalize_vert, vgrid(d, d.nv), dim3(32, 8), 0, d, (float)(1.0 / h));
  LAUNCHP(KID_FIN_ENV, s, k_finalize_env, eblocks32(d), 32, 0, d);
}
void launch_markers(const Dev& d, float* out, int ncomp, cudaStream_t s) {
  int n = d.E * d.nm;
  float4 t1 = make_float4(d.t1[0], d.t1[1], d.t1[2], 0), t2 = make_float4(d.t2[0], d.t2[1], d.t2[2], 0),
         nn = make_float4(d.nrm[0], d.nrm[1], d.nrm[2], 0);
  LAUNCHP(KID_MARKERS, s, k_markers, (n + 255) / 256, 256, 0, d, out, ncomp, t1, t2, nn);
}
void launch_marker_sqerr(const Dev& d, const float* ref, double* acc, int ncomp, cudaStream_t s) {
  float4 t1 = make_float4(d.t1[0], d.t1[1], d.t1[2], 0), t2 = make_float4(d.t2[0], d.t2[1], d.t2[2], 0),
         nn = make_float4(d.nrm[0], d.nrm[1], d.nrm[2], 0);
  LAUNCHP(KID_MARKERS, s, k_marker_sqerr, d.E, 128, 0, d, ref, acc, ncomp, t1, t2, nn);
}
void launch_reset(const Dev& d, const unsigned char* mask, const float* poses, cudaStream_t s) {
  LAUNCHP(KID_OTHER, s, k_reset_env, eblocks(d), 128, 0, d, mask, poses);
  LAUNCHP(KID_OTHER, s, k_reset_vert, vgrid(d, d.nv), dim3(32, 8), 0, d, mask);
}
void launch_status(const Dev& d, int* iters, float* pg, unsigned* flags, cudaStream_t s) {
  LAUNCHP(KID_OTHER, s, k_status, eblocks(d), 128, 0, d, iters, pg, flags);
}
void launch_stats(const Dev& d, int4* out, cudaStream_t s) {
  LAUNCHP(KID_OTHER, s, k_stats, eblocks(d), 128, 0, d, out);
}
void launch_any_active(const Dev& d, int* out, cudaStream_t s) {
  LAUNCHP(KID_OTHER, s, k_any_active, eblocks(d), 128, 0, d, out);
}
void launch_loop_ctl(const Dev& d, cudaGraphConditionalHandle h, int* ctr, int limit, cudaStream_t s) {
  LAUNCHP(KID_OTHER, s, k_loop_ctl, 1, 1024, 0, d, h, ctr, limit);
}
void launch_write_words(const Dev& d, uint64_t* dst, const uint64_t* words, int n, cudaStream_t s) {
  (void)d;
  Words8 v{};
  for (int i = 0; i < n && i < 8; ++i) v.w[i] = words[i];
  LAUNCHP(KID_OTHER, s, k_write_words, 1, 32, 0, dst, v, n);
}
void launch_debug_broadphase(const Dev& d, double r, unsigned long long* out, int* cnt, int cap, cudaStream_t s) {
  int ntot = d.nsv + d.nse + d.nst;
  LAUNCHP(KID_BROADPHASE, s, k_broadphase, dim3((ntot + 127) / 128, d.E), 128, 0, d, r, out, cnt, cap);
}
constexpr int kContactSmemCap = 160 * 1024;  // staged contact kernels: largest dynamic shared size
int contact_smem_bytes(int nsv, int niv) {
  // classify and the staged curvature pass: [nsv + niv] float4
  size_t b = sizeof(float4) * (size_t)(nsv + niv);
  return b <= (size_t)kContactSmemCap ? (int)b : 0;
}
void kernels_init(int contact_smem) {
  cudaFuncSetAttribute(k_sort_anchors, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  // the attribute belongs to the kernel, not to a simulator: several simulators in one
  // process (different meshes) share it, so it is set to the cap contact_smem_bytes
  // enforces rather than to this simulator's size (occupancy follows the launch size)
  (void)contact_smem;
  cudaFuncSetAttribute(k_contact_classify_staged<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kContactSmemCap);
  cudaFuncSetAttribute(k_contact_classify_staged<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kContactSmemCap);
  cudaFuncSetAttribute(k_contact_classify_staged<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kContactSmemCap);
  cudaFuncSetAttribute(k_contact_classify_staged<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kContactSmemCap);
  cudaFuncSetAttribute(k_contact_curv_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, kContactSmemCap);
  cudaFuncSetAttribute(k_elem_curv_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, kTiledCurvSmem);
}

}  // namespace tac
