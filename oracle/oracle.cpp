// oracle.cpp — plain, slow, fp64 CPU oracle of the Tac2Real PNCG-IPC hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code,
// header, helper or constant generator with the CUDA path (paper_2603_28475_b200/csrc).
//
// What it computes (citations: P:L = /root/reference/PAPER.md line L, S:L = SPEC.md):
//   * the incremental potential of Supp. Eq. (ipc_energy)
//       E(x) = 1/2 (x-x^)^T M (x-x^) + h^2 Psi(x) + kappa sum_k b(d_k) + D(x)
//     with x^ = x^t + h v^t, friction D of Eq. (friction_energy) P:436-446,
//     plus the rigid-indenter pose penalty of DESIGN.md reading R18;
//   * its minimisation by the preconditioned Dai-Kou NCG of Eq. (dk_direction),
//     P:450-457, with the step size of Eq. (step_size), extended by the
//     readings R14 (Armijo) and R15 (conservative CCD bound) of DESIGN.md;
//   * the marker displacement field.
// Every function cites the passage it follows.  Where the paper is silent the
// DESIGN.md reading number (R#) is given.  There is no blocking, fusion or
// reordering: loops run over elements / pairs / vertices in index order.
//
// Parity status: every part is pinned by tests/test_oracle_*.py except the
// absolute physical magnitudes of a whole step ("parity unpinned" against the
// paper: the paper prints no worked solver values).
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -shared -fPIC oracle.cpp -o liboracle.so -lpthread

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <set>
#include <thread>
#include <tuple>
#include <vector>

namespace {

typedef std::array<double, 3> V3;
typedef std::array<double, 9> M3;  // row-major

const double INF = std::numeric_limits<double>::infinity();

V3 add(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
V3 sub(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
V3 scl(double s, const V3& a) { return {s * a[0], s * a[1], s * a[2]}; }
double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
double norm(const V3& a) { return std::sqrt(dot(a, a)); }
V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
V3 matvec(const M3& A, const V3& x) {
  return {A[0] * x[0] + A[1] * x[1] + A[2] * x[2], A[3] * x[0] + A[4] * x[1] + A[5] * x[2],
          A[6] * x[0] + A[7] * x[1] + A[8] * x[2]};
}
M3 matmul(const M3& A, const M3& B) {
  M3 C{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k) C[3 * i + j] += A[3 * i + k] * B[3 * k + j];
  return C;
}
M3 transpose(const M3& A) { return {A[0], A[3], A[6], A[1], A[4], A[7], A[2], A[5], A[8]}; }
double det3(const M3& A) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
         A[2] * (A[3] * A[7] - A[4] * A[6]);
}
// cofactor matrix: cof(A) = det(A) A^{-T}; (cof A)_ij = dJ/dA_ij
M3 cof3(const M3& A) {
  return {A[4] * A[8] - A[5] * A[7], A[5] * A[6] - A[3] * A[8], A[3] * A[7] - A[4] * A[6],
          A[2] * A[7] - A[1] * A[8], A[0] * A[8] - A[2] * A[6], A[1] * A[6] - A[0] * A[7],
          A[1] * A[5] - A[2] * A[4], A[2] * A[3] - A[0] * A[5], A[0] * A[4] - A[1] * A[3]};
}
M3 inv3(const M3& A) {
  M3 C = cof3(A);
  double d = det3(A);
  M3 R = transpose(C);
  for (double& x : R) x /= d;
  return R;
}
M3 skew(const V3& w) { return {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0}; }

// ---- SO(3) (R18: rigid indenter pose, left-trivialised rotation) ----
M3 quat_to_R(const double* q7) {  // q7 = (t, q_w, q_x, q_y, q_z); q normalised in fp64 first
  double w = q7[3], x = q7[4], y = q7[5], z = q7[6];
  double n = std::sqrt(w * w + x * x + y * y + z * z);
  w /= n; x /= n; y /= n; z /= n;
  return {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
          2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
          2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
}
M3 so3_exp(const V3& w) {  // Rodrigues
  double th = norm(w);
  M3 K = skew(w);
  M3 K2 = matmul(K, K);
  double a, b;
  if (th < 1e-8) { a = 1 - th * th / 6; b = 0.5 - th * th / 24; }
  else { a = std::sin(th) / th; b = (1 - std::cos(th)) / (th * th); }
  M3 R{1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int i = 0; i < 9; ++i) R[i] += a * K[i] + b * K2[i];
  return R;
}
V3 so3_log(const M3& R) {
  double tr = R[0] + R[4] + R[8];
  double c = std::max(-1.0, std::min(1.0, (tr - 1) / 2));
  double th = std::acos(c);
  V3 v = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
  if (th < 1e-6) return scl(0.5 * (1 + th * th / 6), v);
  if (M_PI - th < 1e-6) {  // near pi: axis from the symmetric part
    int i = (R[0] >= R[4] && R[0] >= R[8]) ? 0 : (R[4] >= R[8] ? 1 : 2);
    V3 a{};
    a[i] = std::sqrt(std::max(0.0, (R[4 * i] + 1) / 2));
    for (int j = 0; j < 3; ++j)
      if (j != i) a[j] = (R[3 * i + j] + R[3 * j + i]) / (4 * a[i]);
    double n = norm(a);
    return scl(th / n, a);
  }
  return scl(th / (2 * std::sin(th)), v);
}

// ---- barrier; formula per DESIGN.md R3 (IPC barrier on unsquared d) ----
double barrier_b(double d, double dh) {
  if (d >= dh) return 0.0;
  return -(d - dh) * (d - dh) * std::log(d / dh);
}
double barrier_db(double d, double dh) {
  if (d >= dh) return 0.0;
  return -2 * (d - dh) * std::log(d / dh) - (d - dh) * (d - dh) / d;
}
double barrier_ddb(double d, double dh) {
  if (d >= dh) return 0.0;
  return -2 * std::log(d / dh) - 4 * (d - dh) / d + (d - dh) * (d - dh) / (d * d);
}
// ---- friction mollifier, Supp. Eq. (friction_mollifier) P:443 ----
double moll_f(double s, double eps) {
  if (s >= eps) return s;
  return -s * s * s / (3 * eps * eps) + s * s / eps + eps / 3;
}
double moll_df(double s, double eps) {
  if (s >= eps) return 1.0;
  return -s * s / (eps * eps) + 2 * s / eps;
}
double moll_f1(double s, double eps) {  // f'(s)/s, finite at s=0
  if (s >= eps) return 1.0 / s;
  return -s / (eps * eps) + 2 / eps;
}

// J_l(phi)^-T x for the SO(3) left Jacobian: J_l^-1 = I - [phi]/2 + c(t) [phi]^2,
// c(t) = (1 - (t/2) cot(t/2)) / t^2 (-> 1/12), t = |phi|; its transpose flips the [phi] term
V3 so3_jl_inv_T(const V3& phi, const V3& x) {
  double t = norm(phi);
  double c = t < 1e-4 ? 1.0 / 12.0 + t * t / 720.0 : (1.0 - 0.5 * t / std::tan(0.5 * t)) / (t * t);
  V3 px = cross(phi, x);
  return add(add(x, scl(0.5, px)), scl(c, cross(phi, px)));
}

// ---- edge-edge mollifier (R30; IPC's parallel-edge treatment) ----
// c = |e_a x e_b|^2, eps_x = 1e-3 |E_a|^2 |E_b|^2 (rest edges); m(c) = -c^2/eps^2 + 2c/eps for
// c < eps, else 1 (C^1 at eps); the EE barrier becomes m(c) kappa b(d)
struct Moll {
  double m = 1, dm = 0;  // m(c), m'(c)
  V3 dc[4] = {};         // dc/dz_k for the corners (a0, a1, b0, b1)
};
Moll ee_mollifier(const V3 z[4], double La2, double Lb2) {
  Moll M;
  V3 ea = sub(z[1], z[0]), eb = sub(z[3], z[2]);
  V3 w = cross(ea, eb);
  double c = dot(w, w), eps = 1e-3 * La2 * Lb2;
  V3 ga = scl(2.0, cross(eb, w)), gb = scl(2.0, cross(w, ea));  // dc/de_a, dc/de_b
  M.dc[0] = scl(-1.0, ga); M.dc[1] = ga; M.dc[2] = scl(-1.0, gb); M.dc[3] = gb;
  if (c < eps) {
    M.m = (2.0 - c / eps) * c / eps;
    M.dm = (2.0 - 2.0 * c / eps) / eps;
  }
  return M;
}
// ---- force-capped pose spring (R18) ----
double huber(double r, double k, double cap) {
  double rho = cap / k;
  return r <= rho ? 0.5 * k * r * r : cap * (r - 0.5 * rho);
}
double huber_w(double r, double k, double cap) {  // psi'(r)/r: gradient = w * delta, GN curvature = w
  double rho = cap / k;
  return r <= rho ? k : cap / r;
}

// ---- primitive distances ("distance between a contact primitive pair") ----
// Result: d = |r|, r = sum_i w[i] z_i over the 4 corners (A-side weights >= 0,
// B-side weights <= 0).  The minimum of a convex quadratic over a simplex pair
// is at the interior critical point or on the boundary: we take the interior
// solution when it is valid, else the point-edge distances in a fixed order.
struct Dist {
  double d;
  double w[4];
  int n;  // 3 corners for point-edge (internal), 4 otherwise
};
// point p vs segment (a,b): closest point a + t(b-a)
double pe_param(const V3& p, const V3& a, const V3& b) {
  V3 e = sub(b, a);
  double t = dot(sub(p, a), e) / dot(e, e);
  return std::max(0.0, std::min(1.0, t));
}
// point-triangle: corners (p, t0, t1, t2), weights (1, -b0, -b1, -b2)
Dist dist_pt(const V3& p, const V3& t0, const V3& t1, const V3& t2) {
  V3 e1 = sub(t1, t0), e2 = sub(t2, t0), q = sub(p, t0);
  double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2);
  double r1 = dot(q, e1), r2 = dot(q, e2);
  double det = a11 * a22 - a12 * a12;
  double s = (a22 * r1 - a12 * r2) / det, t = (a11 * r2 - a12 * r1) / det;
  Dist best;
  best.d = INF;
  if (s >= 0 && t >= 0 && s + t <= 1) {
    V3 c = add(t0, add(scl(s, e1), scl(t, e2)));
    best.d = norm(sub(p, c));
    best.w[0] = 1; best.w[1] = -(1 - s - t); best.w[2] = -s; best.w[3] = -t;
    best.n = 4;
    return best;
  }
  const V3* T[3] = {&t0, &t1, &t2};
  for (int k = 0; k < 3; ++k) {  // edges (t0,t1), (t1,t2), (t2,t0); first minimum wins
    int i = k, j = (k + 1) % 3;
    double u = pe_param(p, *T[i], *T[j]);
    V3 c = add(scl(1 - u, *T[i]), scl(u, *T[j]));
    double d = norm(sub(p, c));
    if (d < best.d) {
      best.d = d;
      best.w[0] = 1; best.w[1] = best.w[2] = best.w[3] = 0;
      best.w[1 + i] = -(1 - u);
      best.w[1 + j] = -u;
      best.n = 4;
    }
  }
  return best;
}
// edge-edge: corners (a0, a1, b0, b1), weights (1-s, s, -(1-t), -t)
Dist dist_ee(const V3& a0, const V3& a1, const V3& b0, const V3& b1) {
  V3 d1 = sub(a1, a0), d2 = sub(b1, b0), r = sub(a0, b0);
  double a = dot(d1, d1), e = dot(d2, d2), b = dot(d1, d2), c = dot(d1, r), f = dot(d2, r);
  double den = a * e - b * b;
  Dist best;
  best.d = INF;
  best.n = 4;
  if (den > 1e-12 * a * e) {  // non-parallel: interior critical point
    double s = (b * f - c * e) / den, t = (a * f - b * c) / den;
    if (s > 0 && s < 1 && t > 0 && t < 1) {
      V3 pa = add(a0, scl(s, d1)), pb = add(b0, scl(t, d2));
      best.d = norm(sub(pa, pb));
      best.w[0] = 1 - s; best.w[1] = s; best.w[2] = -(1 - t); best.w[3] = -t;
      return best;
    }
  }
  // boundary: a0 vs B, a1 vs B, b0 vs A, b1 vs A (R25), first minimum wins
  {
    double t = pe_param(a0, b0, b1);
    double d = norm(sub(a0, add(scl(1 - t, b0), scl(t, b1))));
    if (d < best.d) { best.d = d; best.w[0] = 1; best.w[1] = 0; best.w[2] = -(1 - t); best.w[3] = -t; }
  }
  {
    double t = pe_param(a1, b0, b1);
    double d = norm(sub(a1, add(scl(1 - t, b0), scl(t, b1))));
    if (d < best.d) { best.d = d; best.w[0] = 0; best.w[1] = 1; best.w[2] = -(1 - t); best.w[3] = -t; }
  }
  {
    double s = pe_param(b0, a0, a1);
    double d = norm(sub(add(scl(1 - s, a0), scl(s, a1)), b0));
    if (d < best.d) { best.d = d; best.w[0] = 1 - s; best.w[1] = s; best.w[2] = -1; best.w[3] = 0; }
  }
  {
    double s = pe_param(b1, a0, a1);
    double d = norm(sub(add(scl(1 - s, a0), scl(s, a1)), b1));
    if (d < best.d) { best.d = d; best.w[0] = 1 - s; best.w[1] = s; best.w[2] = 0; best.w[3] = -1; }
  }
  return best;
}

// ---------------------------------------------------------------------------
// static problem data
// ---------------------------------------------------------------------------
enum Kind { PT_GI = 0, PT_IG = 1, EE = 2 };  // (gel vert, ind tri) (ind vert, gel tri) (gel edge, ind edge)

struct Pair {
  int kind, a, b;  // primitive ids: a on the first side, b on the second side (see Kind)
  bool operator<(const Pair& o) const { return std::tie(kind, a, b) < std::tie(o.kind, o.a, o.b); }
};

struct Anchor {  // friction anchor frozen at step start (R7)
  Pair pr;
  double w[4];   // frozen closest-point weights
  V3 z0[4];      // corner positions at step start
  V3 t1, t2;     // tangent basis (T_k), orthogonal to the step-start normal
  double lam;    // lambda_k = -kappa b'(d_k(x^t)) >= 0
};

struct Problem {
  int nv, nt;
  std::vector<V3> X;
  std::vector<std::array<int, 4>> tets;
  std::vector<char> fixed;
  std::vector<std::array<V3, 4>> bvec;  // b_0..b_3 per tet (rows of Dm^-1; b_0 = -sum)
  std::vector<double> vol;              // V_e
  std::vector<double> mass;             // lumped
  // gel surface (boundary faces not entirely fixed)
  std::vector<int> sv;                    // surface vertices
  std::vector<std::array<int, 2>> se;     // surface edges
  std::vector<std::array<int, 3>> st;     // surface triangles
  // indenter (body frame)
  int niv;
  std::vector<V3> Y;
  std::vector<std::array<int, 3>> it;
  std::vector<std::array<int, 2>> ie;
  double rho_max;
  // markers
  int nm;
  std::vector<V3> mk;
  V3 frame[3];
  std::vector<std::array<int, 4>> mk_idx;
  std::vector<std::array<double, 4>> mk_w;
  std::vector<int> mk_tet;
  // material / params
  double mu, lam2;  // mu and lambda' = lambda + mu (R1)
  double rho, mu_f;
  double dhat, kappa_phys, eps_v, tol_x, k_t, k_r, ccd_s, bp_margin, c1, f_max, t_max;
  int max_iters, fixed_iters, beta_rule, precond, max_halvings, stagnation, debug;
  int pose_al;  // augmented-Lagrangian pose enforcement (R29)
  int ee_moll;  // edge-edge parallel mollifier (R30)
  int dedup;    // IPC-toolkit constraint deduplication (R33)
};

struct Env {
  std::vector<V3> u_t, v_t, u;  // displacement at t, velocity at t, current displacement
  V3 c_t, c;
  M3 R_t, R;
  // last-step diagnostics
  int iters = 0, flags = 0;
  double pg = 0, dmin = INF, pose_res = 0;
  V3 lam_t{0, 0, 0}, lam_r{0, 0, 0};  // pose multipliers (R29), 0 without pose_al
  std::vector<std::array<double, 16>> trace;
  bool want_trace = false;
};

struct Oracle {
  Problem P;
  std::vector<Env> env;
  // per-step target pose noise (R27): amplitudes, Philox key, step count
  double noise_t = 0, noise_r = 0;
  uint64_t noise_seed = 0, step_count = 0;
  int64_t env_offset = 0;
  V3 eval_lam_t{0, 0, 0}, eval_lam_r{0, 0, 0};  // multipliers or_eval uses (tests of R29)
};

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2,
// 3", SC'11): 10 rounds of (hi, lo) = M * x products with key bumps by the Weyl constants
// ---------------------------------------------------------------------------
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]}, k[2] = {key_in[0], key_in[1]};
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k[0] += W0; k[1] += W1; }
    const uint64_t p0 = (uint64_t)M0 * c[0], p1 = (uint64_t)M1 * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k[0], n1 = lo1, n2 = hi0 ^ c[3] ^ k[1], n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
  for (int i = 0; i < 4; ++i) out[i] = c[i];
}
// uniform on (-1, 1) from the top 24 bits (exact in fp32 and fp64)
double unit_sym(uint32_t x) { return ((double)(x >> 8) + 0.5) * (2.0 / 16777216.0) - 1.0; }
// R27: target of env `env` at step `step`: c_s += s_t (u0, u1, u2), R_s <- exp([s_r (u3, u4, u5)]) R_s
// with u from Philox4x32-10(key = seed, counter = (env, step_lo, step_hi, 0 / 1))
void perturb_target(uint64_t seed, uint64_t step, uint64_t env, double s_t, double s_r, V3* cs, M3* Rs) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t a[4], b[4];
  const uint32_t c0[4] = {(uint32_t)env, (uint32_t)step, (uint32_t)(step >> 32), 0u};
  const uint32_t c1[4] = {(uint32_t)env, (uint32_t)step, (uint32_t)(step >> 32), 1u};
  philox4x32_10(c0, key, a);
  philox4x32_10(c1, key, b);
  const double u[6] = {unit_sym(a[0]), unit_sym(a[1]), unit_sym(a[2]), unit_sym(a[3]), unit_sym(b[0]), unit_sym(b[1])};
  *cs = add(*cs, V3{s_t * u[0], s_t * u[1], s_t * u[2]});
  *Rs = matmul(so3_exp(V3{s_r * u[3], s_r * u[4], s_r * u[5]}), *Rs);
}

// ---------------------------------------------------------------------------
// setup (DESIGN.md §Oracle "precompute")
// ---------------------------------------------------------------------------
void precompute(Problem& P) {
  P.bvec.resize(P.nt);
  P.vol.resize(P.nt);
  P.mass.assign(P.nv, 0.0);
  for (int e = 0; e < P.nt; ++e) {
    const auto& t = P.tets[e];
    V3 d1 = sub(P.X[t[1]], P.X[t[0]]), d2 = sub(P.X[t[2]], P.X[t[0]]), d3 = sub(P.X[t[3]], P.X[t[0]]);
    M3 Dm = {d1[0], d2[0], d3[0], d1[1], d2[1], d3[1], d1[2], d2[2], d3[2]};  // columns = edges
    P.vol[e] = det3(Dm) / 6.0;
    M3 Bi = inv3(Dm);
    for (int k = 1; k <= 3; ++k) P.bvec[e][k] = {Bi[3 * (k - 1)], Bi[3 * (k - 1) + 1], Bi[3 * (k - 1) + 2]};
    P.bvec[e][0] = scl(-1.0, add(P.bvec[e][1], add(P.bvec[e][2], P.bvec[e][3])));
    for (int k = 0; k < 4; ++k) P.mass[t[k]] += P.rho * P.vol[e] / 4.0;  // lumped mass
  }
  // boundary faces: faces appearing in exactly one tet; drop all-fixed faces (R21)
  std::map<std::array<int, 3>, int> cnt;
  for (const auto& t : P.tets) {
    int f[4][3] = {{t[1], t[2], t[3]}, {t[0], t[2], t[3]}, {t[0], t[1], t[3]}, {t[0], t[1], t[2]}};
    for (auto& ff : f) {
      std::array<int, 3> k = {ff[0], ff[1], ff[2]};
      std::sort(k.begin(), k.end());
      cnt[k]++;
    }
  }
  std::set<int> sv;
  std::set<std::array<int, 2>> se;
  for (const auto& kv : cnt) {
    if (kv.second != 1) continue;
    const auto& k = kv.first;
    if (P.fixed[k[0]] && P.fixed[k[1]] && P.fixed[k[2]]) continue;
    P.st.push_back(k);
    for (int i = 0; i < 3; ++i) {
      sv.insert(k[i]);
      std::array<int, 2> e = {std::min(k[i], k[(i + 1) % 3]), std::max(k[i], k[(i + 1) % 3])};
      se.insert(e);
    }
  }
  P.sv.assign(sv.begin(), sv.end());
  P.se.assign(se.begin(), se.end());
  std::set<std::array<int, 2>> ie;
  for (const auto& t : P.it)
    for (int i = 0; i < 3; ++i) ie.insert({std::min(t[i], t[(i + 1) % 3]), std::max(t[i], t[(i + 1) % 3])});
  P.ie.assign(ie.begin(), ie.end());
  P.rho_max = 0;
  for (const auto& y : P.Y) P.rho_max = std::max(P.rho_max, norm(y));
}

// markers: barycentric weights of the rest tet containing the marker (R22,
// the paper's weighted interpolation over k = 4 nodes); lowest qualifying tet wins.
int locate_markers_bary(Problem& P) {
  P.mk_idx.resize(P.nm);
  P.mk_w.resize(P.nm);
  P.mk_tet.assign(P.nm, -1);
  for (int m = 0; m < P.nm; ++m) {
    for (int e = 0; e < P.nt; ++e) {
      const auto& t = P.tets[e];
      V3 d1 = sub(P.X[t[1]], P.X[t[0]]), d2 = sub(P.X[t[2]], P.X[t[0]]), d3 = sub(P.X[t[3]], P.X[t[0]]);
      M3 Dm = {d1[0], d2[0], d3[0], d1[1], d2[1], d3[1], d1[2], d2[2], d3[2]};
      V3 l = matvec(inv3(Dm), sub(P.mk[m], P.X[t[0]]));
      double b[4] = {1 - l[0] - l[1] - l[2], l[0], l[1], l[2]};
      if (b[0] >= -1e-12 && b[1] >= -1e-12 && b[2] >= -1e-12 && b[3] >= -1e-12) {
        double s = 0;
        for (double& x : b) { x = std::max(0.0, x); s += x; }
        for (int k = 0; k < 4; ++k) { P.mk_idx[m][k] = t[k]; P.mk_w[m][k] = b[k] / s; }
        P.mk_tet[m] = e;
        break;
      }
    }
    if (P.mk_tet[m] < 0) return 2;  // marker outside the mesh -> invalid input
  }
  return 0;
}
// kNN option ("k-nearest neighbor"): k nearest surface vertices, inverse-distance weights
int locate_markers_knn(Problem& P, int k) {
  P.mk_idx.resize(P.nm);
  P.mk_w.resize(P.nm);
  P.mk_tet.assign(P.nm, -1);
  if (k < 1 || k > 4 || (int)P.sv.size() < k) return 2;
  for (int m = 0; m < P.nm; ++m) {
    std::vector<std::pair<double, int>> dv;
    for (int v : P.sv) dv.push_back({norm(sub(P.X[v], P.mk[m])), v});
    std::sort(dv.begin(), dv.end());  // ties -> lower node id
    for (int j = 0; j < 4; ++j) { P.mk_idx[m][j] = dv[0].second; P.mk_w[m][j] = 0; }
    if (dv[0].first == 0) { P.mk_w[m][0] = 1; continue; }
    double s = 0;
    for (int j = 0; j < k; ++j) s += 1 / dv[j].first;
    for (int j = 0; j < k; ++j) { P.mk_idx[m][j] = dv[j].second; P.mk_w[m][j] = (1 / dv[j].first) / s; }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// state helpers
// ---------------------------------------------------------------------------
struct State {  // one iterate: gel displacements + rigid pose
  std::vector<V3> u;
  V3 c;
  M3 R;
};
struct Grad {  // gradient / diagonal blocks; rigid DOF = (c, theta)
  std::vector<V3> g;
  std::vector<M3> D;
  V3 gc, gth;
  M3 Dc, Dth;
};

V3 gel_pos(const Problem& P, const State& s, int v) { return add(P.X[v], s.u[v]); }
V3 ind_pos(const Problem& P, const State& s, int j) { return add(matvec(s.R, P.Y[j]), s.c); }

// corners of a pair: (is_indenter, vertex id) x 4 (PT uses 4 corners, EE 4 corners)
// rest squared lengths of an EE pair's gel edge (corners 0, 1) and indenter edge (2, 3)
void ee_rest(const Problem& P, const int ci[4], double* La2, double* Lb2) {
  V3 a = sub(P.X[ci[1]], P.X[ci[0]]), b = sub(P.Y[ci[3]], P.Y[ci[2]]);
  *La2 = dot(a, a);
  *Lb2 = dot(b, b);
}

void pair_corners(const Problem& P, const Pair& pr, int ci[4], bool ind[4]) {
  if (pr.kind == PT_GI) {
    ci[0] = P.sv[pr.a]; ind[0] = false;
    for (int k = 0; k < 3; ++k) { ci[1 + k] = P.it[pr.b][k]; ind[1 + k] = true; }
  } else if (pr.kind == PT_IG) {
    ci[0] = pr.a; ind[0] = true;
    for (int k = 0; k < 3; ++k) { ci[1 + k] = P.st[pr.b][k]; ind[1 + k] = false; }
  } else {
    ci[0] = P.se[pr.a][0]; ci[1] = P.se[pr.a][1]; ind[0] = ind[1] = false;
    ci[2] = P.ie[pr.b][0]; ci[3] = P.ie[pr.b][1]; ind[2] = ind[3] = true;
  }
}
V3 corner_pos(const Problem& P, const State& s, int c, bool ind) { return ind ? ind_pos(P, s, c) : gel_pos(P, s, c); }

Dist pair_dist(const Problem& P, const State& s, const Pair& pr) {
  int ci[4];
  bool ind[4];
  pair_corners(P, pr, ci, ind);
  V3 z[4];
  for (int k = 0; k < 4; ++k) z[k] = corner_pos(P, s, ci[k], ind[k]);
  if (pr.kind == EE) return dist_ee(z[0], z[1], z[2], z[3]);
  return dist_pt(z[0], z[1], z[2], z[3]);
}

// ---------------------------------------------------------------------------
// IPC-toolkit constraint deduplication (R33): a pair's constraint is
// identified by its closest features -- the corners with a non-zero closest-point weight on
// each side (gel vertex / edge / face, indenter vertex / edge / face).  A point-edge or
// point-point constraint (one side a single vertex, the other at most an edge) is realised by
// several primitive pairs (the triangles and edges around the feature); it is counted once.
// Point-face and edge-edge-interior constraints belong to one pair only.
// ---------------------------------------------------------------------------
typedef std::array<int, 5> CKey;  // (gel ids sorted, -1 padded) x 2, (indenter ids sorted) x 2, 0
bool dedup_key(const Problem& P, const Pair& pr, const Dist& D, CKey* key) {
  int ci[4];
  bool ind[4];
  pair_corners(P, pr, ci, ind);
  std::vector<int> g, y;
  for (int k = 0; k < 4; ++k)
    if (D.w[k] != 0.0) (ind[k] ? y : g).push_back(ci[k]);
  if (g.size() > 2 || y.size() > 2 || (g.size() == 2 && y.size() == 2)) return false;  // face / edge-edge
  std::sort(g.begin(), g.end());
  std::sort(y.begin(), y.end());
  *key = {g.size() > 0 ? g[0] : -1, g.size() > 1 ? g[1] : -1, y.size() > 0 ? y[0] : -1, y.size() > 1 ? y[1] : -1, 0};
  return true;
}
// true if the pair's constraint was already counted (and records it otherwise)
bool dedup_seen(const Problem& P, const Pair& pr, const Dist& D, std::set<CKey>* seen, bool* interior_ee) {
  CKey key;
  const bool shared = dedup_key(P, pr, D, &key);
  if (interior_ee) *interior_ee = !shared && pr.kind == EE;
  if (!P.dedup || !shared) return false;
  return !seen->insert(key).second;
}

// ---------------------------------------------------------------------------
// broad phase (R16): all (gel vert, ind tri), (ind vert,
// gel tri), (gel edge, ind edge) pairs whose axis-aligned boxes IN THE INDENTER BODY
// FRAME are within r on every axis (complete: a pair at distance <= r has every axis
// gap <= r in any frame).  Brute force O(n m), fp64, no FMA contraction (built with
// -ffp-contract=off) -> the exact predicate the device path must match bit for bit.
// ---------------------------------------------------------------------------
struct Box { double lo[3], hi[3]; };
Box box_of(const V3* z, int n) {
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = z[0][a]; b.hi[a] = z[0][a];
    for (int k = 1; k < n; ++k) { b.lo[a] = std::min(b.lo[a], z[k][a]); b.hi[a] = std::max(b.hi[a], z[k][a]); }
  }
  return b;
}
bool near_boxes(const Box& A, const Box& B, double r) {
  for (int a = 0; a < 3; ++a) {
    if (A.lo[a] > B.hi[a] + r) return false;
    if (B.lo[a] > A.hi[a] + r) return false;
  }
  return true;
}
// gb: gel vertices in the body frame; the indenter boxes come from its rest shape Y
std::vector<Pair> broad_phase(const Problem& P, const std::vector<V3>& gb, double r) {
  const std::vector<V3>& iy = P.Y;
  std::vector<Box> bsv(P.sv.size()), bse(P.se.size()), bst(P.st.size()), biv(P.niv), bie(P.ie.size()), bit(P.it.size());
  for (size_t i = 0; i < P.sv.size(); ++i) bsv[i] = box_of(&gb[P.sv[i]], 1);
  for (size_t i = 0; i < P.se.size(); ++i) { V3 z[2] = {gb[P.se[i][0]], gb[P.se[i][1]]}; bse[i] = box_of(z, 2); }
  for (size_t i = 0; i < P.st.size(); ++i) { V3 z[3] = {gb[P.st[i][0]], gb[P.st[i][1]], gb[P.st[i][2]]}; bst[i] = box_of(z, 3); }
  for (int i = 0; i < P.niv; ++i) biv[i] = box_of(&iy[i], 1);
  for (size_t i = 0; i < P.ie.size(); ++i) { V3 z[2] = {iy[P.ie[i][0]], iy[P.ie[i][1]]}; bie[i] = box_of(z, 2); }
  for (size_t i = 0; i < P.it.size(); ++i) { V3 z[3] = {iy[P.it[i][0]], iy[P.it[i][1]], iy[P.it[i][2]]}; bit[i] = box_of(z, 3); }
  std::vector<Pair> out;
  for (size_t a = 0; a < bsv.size(); ++a)
    for (size_t b = 0; b < bit.size(); ++b)
      if (near_boxes(bsv[a], bit[b], r)) out.push_back({PT_GI, (int)a, (int)b});
  for (size_t a = 0; a < biv.size(); ++a)
    for (size_t b = 0; b < bst.size(); ++b)
      if (near_boxes(biv[a], bst[b], r)) out.push_back({PT_IG, (int)a, (int)b});
  for (size_t a = 0; a < bse.size(); ++a)
    for (size_t b = 0; b < bie.size(); ++b)
      if (near_boxes(bse[a], bie[b], r)) out.push_back({EE, (int)a, (int)b});
  return out;
}
// gel vertices in the body frame: b = R^T (x - c), x = X + u (exact in fp64 for fp32
// inputs), b_a = (R_0a dx_0 + R_1a dx_1) + R_2a dx_2 evaluated left to right
void body_coords(const Problem& P, const State& s, std::vector<V3>& gb) {
  gb.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) {
    V3 x = add(P.X[v], s.u[v]);
    double d0 = x[0] - s.c[0], d1 = x[1] - s.c[1], d2 = x[2] - s.c[2];
    for (int a = 0; a < 3; ++a) {
      double t0 = s.R[a] * d0;
      double t1 = s.R[3 + a] * d1;
      double t2 = s.R[6 + a] * d2;
      gb[v][a] = (t0 + t1) + t2;
    }
  }
}
std::vector<Pair> broad_phase_state(const Problem& P, const State& s, double r) {
  std::vector<V3> gb;
  body_coords(P, s, gb);
  return broad_phase(P, gb, r);
}

// ---------------------------------------------------------------------------
// energy, gradient, diagonal blocks
// ---------------------------------------------------------------------------
struct Step {  // per-step constants
  std::vector<V3> xhat_u;  // u^ = u^t + h v^t
  V3 cs;                   // target c*
  M3 Rs;                   // target R*
  double h, kappa, eps;
  V3 lam_t{0, 0, 0}, lam_r{0, 0, 0};  // pose multipliers of this step (R29)
  std::vector<Anchor> anchors;
};

// Stable Neo-Hookean (R1): Psi = mu/2(|F|^2-3) - mu(J-1) + lambda'/2 (J-1)^2.
// With F = I + G (G = sum_v u_v b_v^T, the displacement gradient; sum_v X_v b_v^T = I):
//   |F|^2 - 3 = 2 tr G + |G|^2,   J - 1 = det(I+G) - 1 = tr G + i2(G) + det G,
// i2 = sum of the principal 2x2 minors of G.  Same function, no 3 - 3 cancellation.
double snh_psi_G(const Problem& P, const M3& G) {
  double trG = G[0] + G[4] + G[8];
  double GG = 0;
  for (double x : G) GG += x * x;
  double i2 = (G[0] * G[4] - G[1] * G[3]) + (G[0] * G[8] - G[2] * G[6]) + (G[4] * G[8] - G[5] * G[7]);
  double Jm1 = trG + i2 + det3(G);
  double Im3 = 2 * trG + GG;
  return P.mu / 2 * Im3 - P.mu * Jm1 + P.lam2 / 2 * Jm1 * Jm1;
}
double snh_psi(const Problem& P, const M3& F) {  // F given (used by the scalar pin)
  M3 G = F;
  G[0] -= 1; G[4] -= 1; G[8] -= 1;
  return snh_psi_G(P, G);
}
M3 disp_gradient(const Problem& P, const std::vector<V3>& u, int e) {  // G = sum_v u_v b_v^T
  M3 G{};
  for (int k = 0; k < 4; ++k) {
    const V3& x = u[P.tets[e][k]];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) G[3 * i + j] += x[i] * P.bvec[e][k][j];
  }
  return G;
}
M3 deformation_gradient(const Problem& P, const std::vector<V3>& u, int e) {  // F = I + G
  M3 F = disp_gradient(P, u, e);
  F[0] += 1; F[4] += 1; F[8] += 1;
  return F;
}
double det_minus_1(const M3& G) {  // det(I + G) - 1
  double trG = G[0] + G[4] + G[8];
  double i2 = (G[0] * G[4] - G[1] * G[3]) + (G[0] * G[8] - G[2] * G[6]) + (G[4] * G[8] - G[5] * G[7]);
  return trG + i2 + det3(G);
}

// barrier + friction contributions of a pair to (value, corner forces, GN diag)
// corner force f_i = dE/dz_i; gel corners -> g_v; indenter corners -> (g_c, g_theta)
void add_corner_force(const Problem& P, const State& s, Grad* G, int c, bool ind, const V3& f) {
  if (!ind) {
    if (!P.fixed[c]) G->g[c] = add(G->g[c], f);
    return;
  }
  V3 arm = sub(ind_pos(P, s, c), s.c);
  G->gc = add(G->gc, f);
  G->gth = add(G->gth, cross(arm, f));
}

// E(x) and optionally g, D, over candidate pairs `C` (O4a-b)
double eval_energy(const Problem& P, const Step& S, const State& s, const std::vector<Pair>& C, Grad* G,
                   double* parts = nullptr) {
  double h2 = S.h * S.h;
  if (G) {
    G->g.assign(P.nv, V3{0, 0, 0});
    G->D.assign(P.nv, M3{});
    G->gc = G->gth = V3{0, 0, 0};
    G->Dc = G->Dth = M3{};
  }
  // inertia 1/2 (x-x^)^T M (x-x^), lumped M
  double Ein = 0;
  for (int v = 0; v < P.nv; ++v) {
    if (P.fixed[v]) continue;
    V3 d = sub(s.u[v], S.xhat_u[v]);
    Ein += 0.5 * P.mass[v] * dot(d, d);
    if (G) {
      G->g[v] = add(G->g[v], scl(P.mass[v], d));
      for (int i = 0; i < 3; ++i) G->D[v][4 * i] += P.mass[v];
    }
  }
  // elasticity h^2 sum_e V_e Psi(F_e), gradient P(F) b_v, exact PSD diag blocks
  double Eel = 0;
  for (int e = 0; e < P.nt; ++e) {
    M3 Gd = disp_gradient(P, s.u, e);
    double w = h2 * P.vol[e];
    Eel += w * snh_psi_G(P, Gd);
    if (!G) continue;
    M3 F = Gd;
    F[0] += 1; F[4] += 1; F[8] += 1;
    double Jm1 = det_minus_1(Gd);
    M3 C = cof3(F);
    M3 PK;  // dPsi/dF = mu F + (lambda'(J-1) - mu) cof F
    for (int i = 0; i < 9; ++i) PK[i] = P.mu * F[i] + (P.lam2 * Jm1 - P.mu) * C[i];
    for (int k = 0; k < 4; ++k) {
      int v = P.tets[e][k];
      if (P.fixed[v]) continue;
      const V3& b = P.bvec[e][k];
      G->g[v] = add(G->g[v], scl(w, matvec(PK, b)));
      // d^2 Psi along dF = delta b^T: mu |b|^2 I + lambda' c c^T, c = cof(F) b (det is linear along a rank-one direction)
      V3 cv = matvec(C, b);
      double bb = dot(b, b);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G->D[v][3 * i + j] += w * ((i == j ? P.mu * bb : 0.0) + P.lam2 * cv[i] * cv[j]);
    }
  }
  // barrier kappa sum_{k in C} b(d_k); with dedup (R33) each constraint once
  double Eb = 0;
  std::set<CKey> seen;
  for (const Pair& pr : C) {
    Dist D = pair_dist(P, s, pr);
    if (!(D.d > 0)) return std::numeric_limits<double>::quiet_NaN();  // infeasible
    if (D.d >= P.dhat) continue;
    bool ee_int = false;
    if (dedup_seen(P, pr, D, &seen, &ee_int)) continue;
    int ci[4];
    bool ind[4];
    pair_corners(P, pr, ci, ind);
    V3 z[4];
    for (int k = 0; k < 4; ++k) z[k] = corner_pos(P, s, ci[k], ind[k]);
    Moll M;  // m = 1 unless the EE mollifier is on (R30; with dedup, edge-edge constraints only)
    if (P.ee_moll && pr.kind == EE && (!P.dedup || ee_int)) {
      double La2, Lb2;
      ee_rest(P, ci, &La2, &Lb2);
      M = ee_mollifier(z, La2, Lb2);
    }
    const double bk = S.kappa * barrier_b(D.d, P.dhat);
    Eb += M.m * bk;
    if (!G) continue;
    V3 r{0, 0, 0};
    for (int k = 0; k < 4; ++k) r = add(r, scl(D.w[k], z[k]));
    V3 n = scl(1.0 / D.d, r);  // dd/dz_k = w_k n
    double db = M.m * S.kappa * barrier_db(D.d, P.dhat), ddb = M.m * S.kappa * barrier_ddb(D.d, P.dhat);
    double sig = 0;  // sum of indenter weights
    V3 rho{0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      // d(m kappa b)/dz_k = m kappa b' w_k n + kappa b m' dc/dz_k (GN blocks keep m kappa b'' only)
      add_corner_force(P, s, G, ci[k], ind[k], add(scl(db * D.w[k], n), scl(bk * M.dm, M.dc[k])));
      if (!ind[k]) {
        if (P.fixed[ci[k]]) continue;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) G->D[ci[k]][3 * i + j] += ddb * D.w[k] * D.w[k] * n[i] * n[j];  // Gauss-Newton (R8)
      } else {
        sig += D.w[k];
        rho = add(rho, scl(D.w[k], sub(z[k], s.c)));
      }
    }
    V3 a = cross(rho, n);  // dd/dtheta
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        G->Dc[3 * i + j] += ddb * sig * sig * n[i] * n[j];
        G->Dth[3 * i + j] += ddb * a[i] * a[j];
      }
  }
  // friction D = mu_f sum lambda_k f(|T_k^T Delta_k|), lagged anchors (R7)
  double Ef = 0;
  for (const Anchor& A : S.anchors) {
    int ci[4];
    bool ind[4];
    pair_corners(P, A.pr, ci, ind);
    V3 z[4];
    V3 Dl{0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      z[k] = corner_pos(P, s, ci[k], ind[k]);
      Dl = add(Dl, scl(A.w[k], sub(z[k], A.z0[k])));
    }
    double tau0 = dot(A.t1, Dl), tau1 = dot(A.t2, Dl);
    double sn = std::sqrt(tau0 * tau0 + tau1 * tau1);
    Ef += P.mu_f * A.lam * moll_f(sn, S.eps);
    if (!G) continue;
    double f1 = P.mu_f * A.lam * moll_f1(sn, S.eps);
    V3 Tt = add(scl(tau0, A.t1), scl(tau1, A.t2));  // T tau
    M3 TT;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) TT[3 * i + j] = A.t1[i] * A.t1[j] + A.t2[i] * A.t2[j];
    double sig = 0;
    V3 rho{0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      add_corner_force(P, s, G, ci[k], ind[k], scl(f1 * A.w[k], Tt));
      if (!ind[k]) {
        if (P.fixed[ci[k]]) continue;
        for (int i = 0; i < 9; ++i) G->D[ci[k]][i] += f1 * A.w[k] * A.w[k] * TT[i];  // GN, PSD (R8)
      } else {
        sig += A.w[k];
        rho = add(rho, scl(A.w[k], sub(z[k], s.c)));
      }
    }
    V3 a1 = cross(rho, A.t1), a2 = cross(rho, A.t2);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        G->Dc[3 * i + j] += f1 * sig * sig * TT[3 * i + j];
        G->Dth[3 * i + j] += f1 * (a1[i] * a1[j] + a2[i] * a2[j]);
      }
  }
  // pose penalty (R18): force-capped quadratic spring towards the target pose,
  // psi(r) = k/2 r^2 for r <= rho, k rho (r - rho/2) beyond, rho = cap/k; scaled by h^2
  V3 dc = sub(s.c, S.cs);
  V3 phi = so3_log(matmul(s.R, transpose(S.Rs)));
  double Ep = h2 * (huber(norm(dc), P.k_t, P.f_max) + huber(norm(phi), P.k_r, P.t_max));
  // augmented Lagrangian (R29): + h^2 (lam_t . dc + lam_r . phi); zero multipliers otherwise
  Ep += h2 * (dot(S.lam_t, dc) + dot(S.lam_r, phi));
  if (G) {
    double wt = huber_w(norm(dc), P.k_t, P.f_max), wr = huber_w(norm(phi), P.k_r, P.t_max);
    G->gc = add(G->gc, scl(h2 * wt, dc));
    G->gth = add(G->gth, scl(h2 * wr, phi));  // exact left-trivialised gradient (App. B)
    // d(lam . phi)/d delta for R <- exp([delta]) R: phi(delta) = log(exp(delta) exp(phi)) has
    // the Jacobian J_l(phi)^-1, so the gradient is J_l(phi)^-T lam (R29)
    G->gc = add(G->gc, scl(h2, S.lam_t));
    G->gth = add(G->gth, scl(h2, so3_jl_inv_T(phi, S.lam_r)));
    for (int i = 0; i < 3; ++i) { G->Dc[4 * i] += h2 * wt; G->Dth[4 * i] += h2 * wr; }
  }
  if (parts) { parts[0] = Ein; parts[1] = Eel; parts[2] = Eb; parts[3] = Ef; parts[4] = Ep; }
  return Ein + Eel + Eb + Ef + Ep;
}

// p^T H p: inertia + exact elastic quadratic form + GN barrier/friction + penalty
double curvature(const Problem& P, const Step& S, const State& s, const std::vector<Pair>& C,
                 const std::vector<V3>& p, const V3& pc, const V3& pth) {
  double h2 = S.h * S.h;
  double q = 0;
  for (int v = 0; v < P.nv; ++v)
    if (!P.fixed[v]) q += P.mass[v] * dot(p[v], p[v]);
  for (int e = 0; e < P.nt; ++e) {
    M3 F = deformation_gradient(P, s.u, e);
    M3 dF{};
    for (int k = 0; k < 4; ++k) {
      const V3& pv = p[P.tets[e][k]];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dF[3 * i + j] += pv[i] * P.bvec[e][k][j];
    }
    double Jm1 = det_minus_1(disp_gradient(P, s.u, e));
    M3 C = cof3(F), CdF = cof3(dF);
    double dd = 0, cd = 0, fc = 0;
    for (int i = 0; i < 9; ++i) { dd += dF[i] * dF[i]; cd += C[i] * dF[i]; fc += F[i] * CdF[i]; }
    // d^2/dt^2 det(F + t dF) at 0 = 2 F : cof(dF)
    q += h2 * P.vol[e] * (P.mu * dd + P.lam2 * cd * cd + (P.lam2 * Jm1 - P.mu) * 2 * fc);
  }
  auto dz = [&](int c, bool ind) -> V3 {
    if (!ind) return p[c];
    return add(pc, cross(pth, sub(ind_pos(P, s, c), s.c)));
  };
  std::set<CKey> seen;
  for (const Pair& pr : C) {
    Dist D = pair_dist(P, s, pr);
    if (D.d >= P.dhat) continue;
    bool ee_int = false;
    if (dedup_seen(P, pr, D, &seen, &ee_int)) continue;  // R33
    int ci[4];
    bool ind[4];
    pair_corners(P, pr, ci, ind);
    V3 r{0, 0, 0}, dr{0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      r = add(r, scl(D.w[k], corner_pos(P, s, ci[k], ind[k])));
      dr = add(dr, scl(D.w[k], dz(ci[k], ind[k])));
    }
    double dn = dot(r, dr) / D.d;
    double m = 1;
    if (P.ee_moll && pr.kind == EE && (!P.dedup || ee_int)) {  // R30: the GN curvature scales with m
      V3 z[4];
      for (int k = 0; k < 4; ++k) z[k] = corner_pos(P, s, ci[k], ind[k]);
      double La2, Lb2;
      ee_rest(P, ci, &La2, &Lb2);
      m = ee_mollifier(z, La2, Lb2).m;
    }
    q += m * S.kappa * barrier_ddb(D.d, P.dhat) * dn * dn;
  }
  for (const Anchor& A : S.anchors) {
    int ci[4];
    bool ind[4];
    pair_corners(P, A.pr, ci, ind);
    V3 Dl{0, 0, 0}, dD{0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      Dl = add(Dl, scl(A.w[k], sub(corner_pos(P, s, ci[k], ind[k]), A.z0[k])));
      dD = add(dD, scl(A.w[k], dz(ci[k], ind[k])));
    }
    double sn = std::hypot(dot(A.t1, Dl), dot(A.t2, Dl));
    double a = dot(A.t1, dD), b = dot(A.t2, dD);
    q += P.mu_f * A.lam * moll_f1(sn, S.eps) * (a * a + b * b);
  }
  V3 dc = sub(s.c, S.cs);
  V3 phi = so3_log(matmul(s.R, transpose(S.Rs)));
  q += h2 * huber_w(norm(dc), P.k_t, P.f_max) * dot(pc, pc) + h2 * huber_w(norm(phi), P.k_r, P.t_max) * dot(pth, pth);
  return q;
}

// ---------------------------------------------------------------------------
// PNCG pieces shared by the IPC step and the quadratic pin
// ---------------------------------------------------------------------------
// Dai-Kou beta, Eq. (dk_direction), written from the per-vector dot products.
// rule 1 = PR+ , 2 = FR (variants), 3 = DK+ : Dai-Kou's truncation
// beta+ = max(beta_DK, eta g_{k+1}^T p_k / |p_k|^2), eta = 0.5 (R28).
double ncg_beta(int rule, double gPy, double yp, double yPy, double pg, double gPg, double gPg_prev, double pp) {
  if (rule == 1) return std::max(0.0, gPy / gPg_prev);
  if (rule == 2) return gPg / gPg_prev;
  double dk = gPy / yp - (yPy / yp) * (pg / yp);
  if (rule == 3) return std::max(dk, 0.5 * pg / pp);
  return dk;
}
// step size, Eq. (step_size): alpha = min(alpha_upper, alpha_bar) (+ alpha_ccd, R15)
double step_alpha_bar(double gp, double pHp) { return pHp > 0 ? -gp / pHp : INF; }
double step_alpha_upper(double dhat, double M) { return M > 0 ? dhat / (2 * M) : INF; }

M3 precond_block(const M3& D, int scalar) {
  if (scalar) return {1 / D[0], 0, 0, 0, 1 / D[4], 0, 0, 0, 1 / D[8]};
  return inv3(D);
}

// ---------------------------------------------------------------------------
// one implicit-Euler step of one environment: SURVEY §8c.2 O1-O5
// ---------------------------------------------------------------------------
struct Vecs {  // search-space vector: gel (V x 3) + rigid (c, theta)
  std::vector<V3> v;
  V3 c, th;
};
double disp_norm(const Problem& P, const Vecs& z) {  // |z|_disp (R11)
  double m = 0;
  for (int v = 0; v < P.nv; ++v)
    if (!P.fixed[v]) m = std::max(m, norm(z.v[v]));
  return std::max(m, norm(z.c) + P.rho_max * norm(z.th));
}
Vecs apply_P(const Problem& P, const Grad& G, const Vecs& g) {
  Vecs r;
  r.v.assign(P.nv, V3{0, 0, 0});
  for (int v = 0; v < P.nv; ++v)
    if (!P.fixed[v]) r.v[v] = matvec(precond_block(G.D[v], P.precond), g.v[v]);
  r.c = matvec(precond_block(G.Dc, P.precond), g.c);
  r.th = matvec(precond_block(G.Dth, P.precond), g.th);
  return r;
}
double vdot(const Problem& P, const Vecs& a, const Vecs& b) {
  double s = 0;
  for (int v = 0; v < P.nv; ++v)
    if (!P.fixed[v]) s += dot(a.v[v], b.v[v]);
  return s + dot(a.c, b.c) + dot(a.th, b.th);
}
Vecs vlin(const Problem& P, double a, const Vecs& x, double b, const Vecs& y) {
  Vecs r;
  r.v.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) r.v[v] = add(scl(a, x.v[v]), scl(b, y.v[v]));
  r.c = add(scl(a, x.c), scl(b, y.c));
  r.th = add(scl(a, x.th), scl(b, y.th));
  return r;
}
State advance(const Problem& P, const State& s, double a, const Vecs& p) {  // O4g
  State r = s;
  for (int v = 0; v < P.nv; ++v)
    if (!P.fixed[v]) r.u[v] = add(s.u[v], scl(a, p.v[v]));
  r.c = add(s.c, scl(a, p.c));
  r.R = matmul(so3_exp(scl(a, p.th)), s.R);
  return r;
}
Vecs to_vecs(const Grad& G) { return Vecs{G.g, G.gc, G.gth}; }

// Conservative step bound over the candidates (R15, "additive-CCD style"
// conservative advancement with a separating plane).  For a pair with closest
// points a* (side A), b* (side B), n = (a*-b*)/d, convexity gives
// n.a >= n.a*, n.b <= n.b* for every point of the two primitives, hence
//   d(alpha) >= min_{i in A} n.a_i(alpha) - max_{j in B} n.b_j(alpha)
//            >= d - alpha * l_n,   l_n = max_A(-n.dz_i) + max_B(n.dz_j) + |p_theta| dhat/4,
// with dz the corner motion per unit alpha (rigid corners: p_c + p_theta x (y-c));
// the last term bounds the rotation's curvature for alpha <= alpha_upper
// (|exp(t[w])r - r - t w x r| <= (t|w|)^2 |r|/2 and alpha |w| rho_max <= dhat/2).
// alpha <= (1-s) d / l_n keeps d(alpha) >= s d.
// Cheap certificates for far pairs: if the world boxes of the two primitives are
// separated along an axis by g >= dhat, that axis is a separating plane with
// separation g (every point of A is beyond every point of B along it); failing that,
// the supporting plane of the pair's primitives (below) is tried.  Either way the same
// bound applies with (g, n) in place of (d, n), and the pair carries no barrier term
// (d >= g >= dhat).  Returns false if neither separates the pair by dhat.
bool axis_separation(const V3* z, int na, double dhat, double* g, V3* n) {
  double best = -INF;
  V3 bn{0, 0, 0};
  for (int a = 0; a < 3; ++a) {
    double loA = INF, hiA = -INF, loB = INF, hiB = -INF;
    for (int k = 0; k < 4; ++k) {
      if (k < na) { loA = std::min(loA, z[k][a]); hiA = std::max(hiA, z[k][a]); }
      else { loB = std::min(loB, z[k][a]); hiB = std::max(hiB, z[k][a]); }
    }
    if (loA - hiB > best) { best = loA - hiB; bn = V3{0, 0, 0}; bn[a] = 1; }   // A above B along +a
    if (loB - hiA > best) { best = loB - hiA; bn = V3{0, 0, 0}; bn[a] = -1; }  // A below B
  }
  if (best < dhat) {
    // primitive-plane certificate: for point-triangle the triangle's supporting plane,
    // for edge-edge the plane spanned by both edge directions (skipped when they are
    // within 1e-3 rad of parallel).  One side lies in the plane and the other is at
    // |m.(z_A - z_B)| / |m| from it, so that plane separates them by that much.
    V3 e1 = sub(z[1], z[0]), e2 = sub(z[3], z[2]), o = sub(z[0], z[2]);
    if (na == 1) { e1 = sub(z[2], z[1]); e2 = sub(z[3], z[1]); o = sub(z[0], z[1]); }
    V3 m = cross(e1, e2);
    double l = norm(m);
    if (l >= 1e-3 * norm(e1) * norm(e2) && l > 0) {
      double sp = std::fabs(dot(m, o)) / l;
      if (sp > best) { best = sp; bn = scl((dot(m, o) >= 0 ? 1.0 : -1.0) / l, m); }
    }
  }
  *g = best;
  *n = bn;
  return best >= dhat;
}
double rel_motion(const Problem& P, const Vecs& p);
// Pairs without a certificate ("near") use their exact closest-point plane.
// All certified ("far") pairs share one bound: each has d(alpha) >= g_i - alpha L_rel
// >= dhat - alpha L_rel (L_rel bounds the relative motion of any gel surface point vs any
// indenter point, see rel_motion), so alpha <= (1-s) dhat / L_rel keeps them >= s dhat
// (R15: the bound depends only on whether a far pair exists, not on its gap).
double alpha_ccd(const Problem& P, const State& s, const std::vector<Pair>& C, const Vecs& p) {
  double pth = norm(p.th);
  double a = INF;
  bool any_far = false;
  for (const Pair& pr : C) {
    int ci[4];
    bool ind[4];
    pair_corners(P, pr, ci, ind);
    V3 z[4], dz[4];
    for (int k = 0; k < 4; ++k) {
      z[k] = corner_pos(P, s, ci[k], ind[k]);
      dz[k] = ind[k] ? add(p.c, cross(p.th, sub(z[k], s.c))) : p.v[ci[k]];
    }
    int na = (pr.kind == EE) ? 2 : 1;
    double g;
    V3 n;
    if (axis_separation(z, na, P.dhat, &g, &n)) {
      any_far = true;
      continue;
    }
    Dist D = pair_dist(P, s, pr);
    if (D.d >= P.dhat) {  // exact distance >= dhat: a far pair like the certified ones (R15)
      any_far = true;
      continue;
    }
    V3 r{0, 0, 0};
    for (int k = 0; k < 4; ++k) r = add(r, scl(D.w[k], z[k]));
    n = scl(1.0 / D.d, r);
    double la = -INF, lb = -INF;
    for (int k = 0; k < 4; ++k) {
      if (k < na) la = std::max(la, -dot(n, dz[k]));
      else lb = std::max(lb, dot(n, dz[k]));
    }
    double l = la + lb + pth * P.dhat / 4;
    if (l > 0) a = std::min(a, (1 - P.ccd_s) * D.d / l);
  }
  double L = rel_motion(P, p);
  if (any_far && L > 0) a = std::min(a, (1 - P.ccd_s) * P.dhat / L);
  return a;
}
// bound on the relative motion of any gel surface point vs any indenter point per unit alpha
double rel_motion(const Problem& P, const Vecs& p) {
  double m = 0;
  for (int v : P.sv) m = std::max(m, norm(sub(p.v[v], p.c)));
  return m + P.rho_max * norm(p.th);
}

// O4e: the search direction, Eq. (dk_direction), with the restarts of R12/R13:
// p = -P g (restart) or -P g + beta p_prev; a non-descent direction restarts
struct Direction {
  Vecs p;
  double beta, gp;  // beta used (0 on a restart), g^T p
  bool restarted;
};
Direction direction(const Problem& P, const Grad& G, const Vecs& g, const Vecs& Pg, double gPg, const Vecs& gprev,
                    const Vecs& pprev, double gPg_prev, bool restart) {
  bool rs = restart;
  double beta = 0;
  if (!rs) {
    Vecs y = vlin(P, 1.0, g, -1.0, gprev);
    Vecs Py = apply_P(P, G, y);  // P_{k+1} y
    double yp = vdot(P, y, pprev);
    double ppn = vdot(P, pprev, pprev);
    double scale = std::sqrt(vdot(P, g, g)) * std::sqrt(ppn);
    if (std::fabs(yp) <= 1e-30 * scale) rs = true;
    else beta = ncg_beta(P.beta_rule, vdot(P, g, Py), yp, vdot(P, y, Py), vdot(P, pprev, g), gPg, gPg_prev, ppn);
    if (!std::isfinite(beta)) rs = true;
  }
  Direction D;
  D.p = rs ? vlin(P, -1.0, Pg, 0.0, Pg) : vlin(P, -1.0, Pg, beta, pprev);
  D.gp = vdot(P, g, D.p);
  D.beta = rs ? 0.0 : beta;
  if (D.gp >= 0) {  // non-descent -> restart
    D.p = vlin(P, -1.0, Pg, 0.0, Pg);
    D.gp = -gPg;
    D.beta = 0;
    rs = true;
  }
  D.restarted = rs;
  return D;
}

// O4f: the step length, Eq. (step_size), alpha = min(alpha_upper, alpha_bar,
// alpha_ccd (R15)); the candidate-list cap of R16 is applied by the caller
struct StepLen {
  double M, a_up, q, a_bar, a_ccd, alpha, Lrel;
};
StepLen step_length(const Problem& P, const Step& S, const State& s, const std::vector<Pair>& C, const Vecs& p,
                    double gp) {
  StepLen L;
  L.M = disp_norm(P, p);
  L.a_up = step_alpha_upper(P.dhat, L.M);
  L.q = curvature(P, S, s, C, p.v, p.c, p.th);
  L.a_bar = step_alpha_bar(gp, L.q);
  L.a_ccd = alpha_ccd(P, s, C, p);
  L.alpha = std::min(L.a_up, std::min(L.a_bar, L.a_ccd));
  if (!std::isfinite(L.alpha)) L.alpha = 0;
  L.Lrel = rel_motion(P, p);
  return L;
}

double brute_dmin(const Problem& P, const State& s) {  // debug: all primitive pairs
  std::vector<Pair> all = broad_phase_state(P, s, INF);
  double m = INF;
  for (const Pair& pr : all) m = std::min(m, pair_dist(P, s, pr).d);
  return m;
}

constexpr double kRebuildAt = 0.75;  // R16: rebuild once the odometer passes this fraction of m_r
enum Flags { F_CONV = 1, F_MAXIT = 2, F_NAN = 4, F_INFEAS = 8, F_LARGE = 16, F_OVERFLOW = 32, F_STAG = 64 };

void build_anchors(const Problem& P, Step& S, const State& s, const std::vector<Pair>& C) {
  S.anchors.clear();
  if (P.mu_f <= 0) return;
  std::set<CKey> seen;
  for (const Pair& pr : C) {
    Dist D = pair_dist(P, s, pr);
    if (!(D.d < P.dhat)) continue;
    bool ee_int = false;
    if (dedup_seen(P, pr, D, &seen, &ee_int)) continue;  // R33: one anchor per constraint
    Anchor A;
    A.pr = pr;
    int ci[4];
    bool ind[4];
    pair_corners(P, pr, ci, ind);
    V3 r{0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      A.w[k] = D.w[k];
      A.z0[k] = corner_pos(P, s, ci[k], ind[k]);
      r = add(r, scl(D.w[k], A.z0[k]));
    }
    V3 n = scl(1.0 / D.d, r);
    int ax = (std::fabs(n[0]) <= std::fabs(n[1]) && std::fabs(n[0]) <= std::fabs(n[2])) ? 0
             : (std::fabs(n[1]) <= std::fabs(n[2]) ? 1 : 2);
    V3 e{0, 0, 0};
    e[ax] = 1;
    V3 t1 = cross(n, e);
    A.t1 = scl(1.0 / norm(t1), t1);
    A.t2 = cross(n, A.t1);
    double m = 1;
    if (P.ee_moll && pr.kind == EE && (!P.dedup || ee_int)) {  // R30: lambda_k of the mollified barrier
      double La2, Lb2;
      ee_rest(P, ci, &La2, &Lb2);
      m = ee_mollifier(A.z0, La2, Lb2).m;
    }
    A.lam = std::max(0.0, -m * S.kappa * barrier_db(D.d, P.dhat));  // lambda_k = -kappa b'(d_k)
    S.anchors.push_back(A);
  }
}

// x0: optional first iterate other than x^t (a feasible state of the same step, e.g. another
// solver's result to be polished); the friction anchors stay those of x^t (R7)
void env_step(const Problem& P, Env& E, const double* target7, double h, const Oracle* O = nullptr,
              int64_t env_id = 0, const State* x0 = nullptr) {
  Step S;
  S.h = h;
  S.kappa = h * h * P.kappa_phys;  // kappa = h^2 kappa_phys (R4)
  S.eps = P.eps_v * h;             // eps = eps_v h
  S.cs = {target7[0], target7[1], target7[2]};
  S.Rs = quat_to_R(target7);
  S.lam_t = E.lam_t;
  S.lam_r = E.lam_r;
  if (O && (O->noise_t != 0 || O->noise_r != 0))
    perturb_target(O->noise_seed, O->step_count, (uint64_t)(env_id + O->env_offset), O->noise_t, O->noise_r, &S.cs,
                   &S.Rs);
  E.flags = 0;
  E.trace.clear();
  // large-motion flag (diagnostic only)
  {
    double dc = norm(sub(S.cs, E.c_t));
    double da = norm(so3_log(matmul(S.Rs, transpose(E.R_t))));
    if (dc > 2e-3 || da > 5 * M_PI / 180) E.flags |= F_LARGE;
  }
  // O1: inertial prediction x^ = x^t + h v^t; fixed vertices stay at X
  S.xhat_u.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) S.xhat_u[v] = P.fixed[v] ? V3{0, 0, 0} : add(E.u_t[v], scl(h, E.v_t[v]));
  // O3: start from the feasible x^t, pose^t (R19)
  State s{E.u_t, E.c_t, E.R_t};
  // O2: broad phase at (x^t, pose^t), friction anchors, S := 0
  const double mr = P.bp_margin, rad = P.dhat + P.bp_margin;
  std::vector<Pair> C = broad_phase_state(P, s, rad);
  build_anchors(P, S, s, C);
  if (x0) {  // another first iterate: candidates at it, anchors from x^t
    s = *x0;
    C = broad_phase_state(P, s, rad);
  }
  double Sacc = 0, Lrel = 0;

  Grad G, Gprev;
  Vecs p, pprev;
  State s_prev = s;
  double E_prev = 0, alpha = 0, gp_prev = 0, gPg_prev = 1;
  bool restart = true, reeval = false;
  int halvings = 0, it = 0;
  double best_pg = INF;
  int best_it = 0;
  bool converged = false, failed = false, last_rejected = false;
  int K = P.fixed_iters > 0 ? P.fixed_iters : P.max_iters;
  for (it = 0; it < K; ++it) {
    // O4b: evaluate
    double parts[5];
    double Ek = eval_energy(P, S, s, C, &G, parts);
    if (!std::isfinite(Ek)) {
      if (it == 0) { failed = true; break; }
    }
    // O4c: Armijo on the incremental potential (R14)
    if (it > 0 && !reeval) {
      bool ok = std::isfinite(Ek) && Ek <= E_prev + P.c1 * alpha * gp_prev;
      if (!ok) {
        ++halvings;
        if (halvings <= P.max_halvings) {
          Sacc += 0.5 * alpha * Lrel;  // odometer: the path back from the rejected trial (R16)
          alpha *= 0.5;
          s = advance(P, s_prev, alpha, p);
        } else {  // give up along p: back to x_k, restart with -P g
          Sacc += alpha * Lrel;
          s = s_prev;
          restart = true;
          reeval = true;
          halvings = 0;
        }
        if (E.want_trace) E.trace.push_back({(double)it, Ek, 0, alpha, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0});
        last_rejected = true;
        continue;
      }
    }
    reeval = false;
    halvings = 0;
    last_rejected = false;
    if (!std::isfinite(Ek)) { failed = true; break; }
    // O4d: convergence on |P g|_disp
    Vecs g = to_vecs(G);
    Vecs Pg = apply_P(P, G, g);
    double pgn = disp_norm(P, Pg);
    if (P.fixed_iters == 0 && pgn <= P.tol_x) { converged = true; E.pg = pgn; break; }
    if (pgn < best_pg * (1 - 1e-3)) { best_pg = pgn; best_it = it; }
    if (P.fixed_iters == 0 && P.stagnation > 0 && it - best_it > P.stagnation) { E.flags |= F_STAG; E.pg = pgn; break; }
    // the last evaluation of the budget: the step ends at this accepted iterate (no new
    // direction, no unevaluated trial is committed)
    if (it == K - 1) { E.pg = pgn; it = K; break; }
    // O4e: direction, Eq. (dk_direction)
    double gPg = vdot(P, g, Pg);
    Direction Dn = direction(P, G, g, Pg, gPg, to_vecs(Gprev), pprev, gPg_prev, restart || it == 0);
    p = Dn.p;
    double gp = Dn.gp, beta = Dn.beta;
    restart = false;
    // O4f: step length, Eq. (step_size) P:459-461 + alpha_ccd (R15)
    StepLen SL = step_length(P, S, s, C, p, gp);
    double M = SL.M, a_up = SL.a_up, q = SL.q, a_bar = SL.a_bar, a_ccd = SL.a_ccd;
    alpha = SL.alpha;
    int rebuilt = 0;
    Lrel = SL.Lrel;
    // R16: the list stays valid while the odometer <= m_r.  A step that would pass m_r is
    // capped at it; the list is rebuilt at the new state once the odometer passes
    // kRebuildAt * m_r (so a later cap never cuts a step below half of alpha_upper)
    if (Lrel > 0 && Sacc + alpha * Lrel > kRebuildAt * mr) {
      if (Sacc + alpha * Lrel > mr) alpha = std::max(0.0, (mr - Sacc) / Lrel);
      rebuilt = 1;
    }
    if (E.want_trace) {
      double dmin = P.debug ? brute_dmin(P, s) : 0;
      E.trace.push_back({(double)it, Ek, 1, alpha, a_up, a_bar, a_ccd, M, pgn, gp, q, (double)rebuilt, dmin,
                         (double)C.size(), (double)S.anchors.size(), beta});
    }
    // O4g: update
    s_prev = s;
    E_prev = Ek;
    Gprev = G;
    pprev = p;
    gp_prev = gp;
    gPg_prev = gPg;
    s = advance(P, s_prev, alpha, p);
    Sacc += alpha * Lrel;
    if (rebuilt) {  // new candidates at the state just reached (O4f)
      C = broad_phase_state(P, s, rad);
      Sacc = 0;
    }
    E.pg = pgn;
  }
  E.iters = it;
  // budget spent on a rejected trial: commit the last accepted iterate x_k, never a trial
  // whose energy was not accepted
  if (!converged && !failed && last_rejected) s = s_prev;
  if (failed) {  // roll back to x^t (SURVEY §5 failure detection)
    E.flags |= F_NAN;
    s = State{E.u_t, E.c_t, E.R_t};
  } else if (converged) E.flags |= F_CONV;
  else if (!(E.flags & F_STAG)) E.flags |= F_MAXIT;
  // O5: v^{t+1} = (x^{t+1} - x^t)/h; store
  for (int v = 0; v < P.nv; ++v) E.v_t[v] = scl(1.0 / h, sub(s.u[v], E.u_t[v]));
  if (failed) for (int v = 0; v < P.nv; ++v) E.v_t[v] = V3{0, 0, 0};
  E.u_t = s.u;
  E.u = s.u;
  E.c_t = s.c;
  E.R_t = s.R;
  E.pose_res = norm(sub(s.c, S.cs)) + P.rho_max * norm(so3_log(matmul(s.R, transpose(S.Rs))));
  if (P.pose_al && !failed) {  // R29: lam += psi'(r) r/|r| at the step's solution (first-order AL update)
    V3 dc = sub(s.c, S.cs);
    V3 phi = so3_log(matmul(s.R, transpose(S.Rs)));
    E.lam_t = add(E.lam_t, scl(huber_w(norm(dc), P.k_t, P.f_max), dc));
    E.lam_r = add(E.lam_r, scl(huber_w(norm(phi), P.k_r, P.t_max), phi));
  }
  if (P.debug) E.dmin = brute_dmin(P, s);
}

}  // namespace

// ===========================================================================
// C API (test infrastructure; ctypes)
// ===========================================================================
extern "C" {

// dparams: dhat, kappa_phys, eps_v, tol_x, k_t, k_r, ccd_s, bp_margin, c1, f_max, t_max
// iparams: max_iters, fixed_iters, beta_rule, precond, max_halvings, stagnation, marker_mode, knn_k, debug,
//          pose_al, ee_mollifier, dedup
void* or_create(int nv, const double* X, int nt, const int* tets, int nfixed, const int* fixed, int niv,
                const double* Y, int nit, const int* itris, int nm, const double* mk, const double* frame9,
                const double* mat4, const double* dparams, const int* iparams, int n_envs, const double* init7,
                int* status) {
  Oracle* O = new Oracle;
  Problem& P = O->P;
  P.nv = nv; P.nt = nt; P.niv = niv; P.nm = nm;
  P.X.resize(nv);
  for (int i = 0; i < nv; ++i) P.X[i] = {X[3 * i], X[3 * i + 1], X[3 * i + 2]};
  P.tets.resize(nt);
  *status = 0;
  for (int e = 0; e < nt; ++e)
    for (int k = 0; k < 4; ++k) {
      P.tets[e][k] = tets[4 * e + k];
      if (tets[4 * e + k] < 0 || tets[4 * e + k] >= nv) *status = 2;
    }
  P.fixed.assign(nv, 0);
  for (int i = 0; i < nfixed; ++i) {
    if (fixed[i] < 0 || fixed[i] >= nv) { *status = 2; continue; }
    P.fixed[fixed[i]] = 1;
  }
  P.Y.resize(niv);
  for (int i = 0; i < niv; ++i) P.Y[i] = {Y[3 * i], Y[3 * i + 1], Y[3 * i + 2]};
  P.it.resize(nit);
  for (int i = 0; i < nit; ++i) for (int k = 0; k < 3; ++k) P.it[i][k] = itris[3 * i + k];
  P.mk.resize(nm);
  for (int i = 0; i < nm; ++i) P.mk[i] = {mk[3 * i], mk[3 * i + 1], mk[3 * i + 2]};
  for (int a = 0; a < 3; ++a) P.frame[a] = {frame9[3 * a], frame9[3 * a + 1], frame9[3 * a + 2]};
  double E = mat4[0], nu = mat4[1];
  P.mu = E / (2 * (1 + nu));
  double lam = E * nu / ((1 + nu) * (1 - 2 * nu));
  P.lam2 = lam + P.mu;
  P.rho = mat4[2]; P.mu_f = mat4[3];
  P.dhat = dparams[0]; P.kappa_phys = dparams[1]; P.eps_v = dparams[2]; P.tol_x = dparams[3];
  P.k_t = dparams[4]; P.k_r = dparams[5]; P.ccd_s = dparams[6]; P.bp_margin = dparams[7]; P.c1 = dparams[8];
  P.f_max = dparams[9]; P.t_max = dparams[10];
  P.max_iters = iparams[0]; P.fixed_iters = iparams[1]; P.beta_rule = iparams[2]; P.precond = iparams[3];
  P.max_halvings = iparams[4]; P.stagnation = iparams[5];
  P.debug = iparams[8];
  P.pose_al = iparams[9];
  P.ee_moll = iparams[10];
  P.dedup = iparams[11];
  if (*status) return O;
  precompute(P);
  for (int e = 0; e < nt; ++e) if (!(P.vol[e] > 0)) *status = 2;
  if (*status) return O;
  if (P.kappa_phys <= 0) {  // default rule (R4): 0.2 E lbar^2 / (12.25 dhat), lbar = mean gel surface edge
    double s = 0;
    for (const auto& e : P.se) s += norm(sub(P.X[e[0]], P.X[e[1]]));
    double lbar = s / P.se.size();
    P.kappa_phys = 0.2 * E * lbar * lbar / (12.25 * P.dhat);
  }
  *status = iparams[6] == 0 ? locate_markers_bary(P) : locate_markers_knn(P, iparams[7]);
  O->env.resize(n_envs);
  for (int e = 0; e < n_envs; ++e) {
    Env& en = O->env[e];
    en.u_t.assign(nv, V3{0, 0, 0});
    en.v_t.assign(nv, V3{0, 0, 0});
    en.u = en.u_t;
    en.c_t = {init7[7 * e], init7[7 * e + 1], init7[7 * e + 2]};
    en.R_t = quat_to_R(init7 + 7 * e);
    en.c = en.c_t;
    en.R = en.R_t;
    State s{en.u_t, en.c_t, en.R_t};
    // an indenter intersecting / touching the gel at its initial pose is invalid input
    for (const Pair& pr : broad_phase_state(P, s, P.dhat))
      if (!(pair_dist(P, s, pr).d > 0)) *status = 2;
  }
  return O;
}
void or_destroy(void* h) { delete (Oracle*)h; }
double or_kappa_phys(void* h) { return ((Oracle*)h)->P.kappa_phys; }
void or_counts(void* h, int* out) {  // surface: verts, edges, tris; indenter edges
  Problem& P = ((Oracle*)h)->P;
  out[0] = P.sv.size(); out[1] = P.se.size(); out[2] = P.st.size(); out[3] = P.ie.size();
}
void or_surface(void* h, int* sv, int* se, int* st, int* ie) {
  Problem& P = ((Oracle*)h)->P;
  for (size_t i = 0; i < P.sv.size(); ++i) sv[i] = P.sv[i];
  for (size_t i = 0; i < P.se.size(); ++i) { se[2 * i] = P.se[i][0]; se[2 * i + 1] = P.se[i][1]; }
  for (size_t i = 0; i < P.st.size(); ++i) for (int k = 0; k < 3; ++k) st[3 * i + k] = P.st[i][k];
  for (size_t i = 0; i < P.ie.size(); ++i) { ie[2 * i] = P.ie[i][0]; ie[2 * i + 1] = P.ie[i][1]; }
}
void or_mass_vol(void* h, double* mass, double* vol) {
  Problem& P = ((Oracle*)h)->P;
  for (int i = 0; i < P.nv; ++i) mass[i] = P.mass[i];
  for (int i = 0; i < P.nt; ++i) vol[i] = P.vol[i];
}
void or_marker_map(void* h, int* tet, int* idx, double* w) {
  Problem& P = ((Oracle*)h)->P;
  for (int m = 0; m < P.nm; ++m) {
    tet[m] = P.mk_tet[m];
    for (int k = 0; k < 4; ++k) { idx[4 * m + k] = P.mk_idx[m][k]; w[4 * m + k] = P.mk_w[m][k]; }
  }
}

// n_threads envs in parallel (one env per thread, each serial), P:180 env independence
void or_step(void* h, const double* targets7, double dt, int n_threads, int env0, int n) {
  Oracle* O = (Oracle*)h;
  if (n <= 0) n = (int)O->env.size() - env0;
  if (n_threads < 1) n_threads = 1;
  std::vector<std::thread> th;
  for (int t = 0; t < n_threads; ++t)
    th.emplace_back([=]() {
      for (int e = env0 + t; e < env0 + n; e += n_threads) env_step(O->P, O->env[e], targets7 + 7 * e, dt, O, e);
    });
  for (auto& x : th) x.join();
  O->step_count += 1;
}
// env `env`'s step from its stored x^t to `target7`, started at the feasible iterate
// (u0, c0, R0) instead of x^t (test hook: polishing another solver's result to decide whether
// it sits at a local minimiser of the same incremental potential)
void or_step_from(void* h, int env, const double* target7, double dt, const double* u0, const double* c0,
                  const double* R0) {
  Oracle* O = (Oracle*)h;
  State x0;
  x0.u.resize(O->P.nv);
  for (int v = 0; v < O->P.nv; ++v) x0.u[v] = {u0[3 * v], u0[3 * v + 1], u0[3 * v + 2]};
  x0.c = {c0[0], c0[1], c0[2]};
  for (int i = 0; i < 9; ++i) x0.R[i] = R0[i];
  env_step(O->P, O->env[env], target7, dt, O, env, &x0);
}
void or_set_pose_noise(void* h, double sigma_t, double sigma_r, uint64_t seed, int64_t env_offset) {
  Oracle* O = (Oracle*)h;
  O->noise_t = sigma_t; O->noise_r = sigma_r; O->noise_seed = seed; O->env_offset = env_offset;
}
void or_philox(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { philox4x32_10(ctr, key, out); }
void or_env_status(void* h, int env, double* out) {  // iters, flags, |Pg|, dmin, pose residual
  Env& E = ((Oracle*)h)->env[env];
  out[0] = E.iters; out[1] = E.flags; out[2] = E.pg; out[3] = E.dmin; out[4] = E.pose_res;
}
void or_get_state(void* h, int env, double* u, double* v, double* c, double* R) {
  Oracle* O = (Oracle*)h;
  Env& E = O->env[env];
  for (int i = 0; i < O->P.nv; ++i) for (int a = 0; a < 3; ++a) { u[3 * i + a] = E.u_t[i][a]; v[3 * i + a] = E.v_t[i][a]; }
  for (int a = 0; a < 3; ++a) c[a] = E.c_t[a];
  for (int a = 0; a < 9; ++a) R[a] = E.R_t[a];
}
void or_set_state(void* h, int env, const double* u, const double* v, const double* c, const double* R) {
  Oracle* O = (Oracle*)h;
  Env& E = O->env[env];
  for (int i = 0; i < O->P.nv; ++i) for (int a = 0; a < 3; ++a) { E.u_t[i][a] = u[3 * i + a]; E.v_t[i][a] = v[3 * i + a]; }
  for (int a = 0; a < 3; ++a) E.c_t[a] = c[a];
  for (int a = 0; a < 9; ++a) E.R_t[a] = R[a];
  E.u = E.u_t; E.c = E.c_t; E.R = E.R_t;
}
void or_set_trace(void* h, int env, int on) { ((Oracle*)h)->env[env].want_trace = on != 0; }
int or_trace(void* h, int env, double* out, int cap) {
  Env& E = ((Oracle*)h)->env[env];
  int n = std::min<int>(cap, E.trace.size());
  for (int i = 0; i < n; ++i) for (int k = 0; k < 16; ++k) out[16 * i + k] = E.trace[i][k];
  return (int)E.trace.size();
}
// marker field: u_m = sum_j w_mj u_j; out[m] = (u_m.t1, u_m.t2 [, u_m.n])
void or_markers(void* h, int env, int ncomp, double* out) {
  Oracle* O = (Oracle*)h;
  Problem& P = O->P;
  Env& E = O->env[env];
  for (int m = 0; m < P.nm; ++m) {
    V3 um{0, 0, 0};
    for (int k = 0; k < 4; ++k) um = add(um, scl(P.mk_w[m][k], E.u_t[P.mk_idx[m][k]]));
    for (int c = 0; c < ncomp; ++c) out[ncomp * m + c] = dot(um, P.frame[c]);
  }
}

// --- debug hooks (kernel-level parity / pins) ---
// Evaluate E, g, D at state (u, c, R) with friction anchors built at (u_t, c_t, R_t) and
// candidates built at (u, c, R); target pose target7; step h.  parts[5] = inertia, elastic,
// barrier, friction, pose.  g [nv*3], D [nv*9], grig [6] = (g_c, g_theta), Drig [18] = (Dc, Dth).
// pose multipliers (R29): those or_eval uses, and an env's current ones (6 = lam_t, lam_r)
void or_set_eval_lambda(void* h, const double* lam6) {
  Oracle* O = (Oracle*)h;
  O->eval_lam_t = {lam6[0], lam6[1], lam6[2]};
  O->eval_lam_r = {lam6[3], lam6[4], lam6[5]};
}
void or_get_lambda(void* h, int env, double* lam6) {
  const Env& E = ((Oracle*)h)->env[env];
  for (int a = 0; a < 3; ++a) { lam6[a] = E.lam_t[a]; lam6[3 + a] = E.lam_r[a]; }
}

double or_eval(void* h, const double* u_t, const double* v_t, const double* ct, const double* Rt, const double* u,
               const double* c, const double* R, const double* target7, double dt, double* parts, double* g,
               double* D, double* grig, double* Drig, int* n_cand, int* n_anchor) {
  Oracle* O = (Oracle*)h;
  Problem& P = O->P;
  Step S;
  S.h = dt;
  S.kappa = dt * dt * P.kappa_phys;
  S.eps = P.eps_v * dt;
  S.cs = {target7[0], target7[1], target7[2]};
  S.Rs = quat_to_R(target7);
  S.lam_t = O->eval_lam_t;
  S.lam_r = O->eval_lam_r;
  S.xhat_u.resize(P.nv);
  State st, s;
  st.u.resize(P.nv);
  s.u.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) {
    V3 a{u_t[3 * v], u_t[3 * v + 1], u_t[3 * v + 2]}, b{v_t[3 * v], v_t[3 * v + 1], v_t[3 * v + 2]};
    st.u[v] = a;
    S.xhat_u[v] = P.fixed[v] ? V3{0, 0, 0} : add(a, scl(dt, b));
    s.u[v] = {u[3 * v], u[3 * v + 1], u[3 * v + 2]};
  }
  st.c = {ct[0], ct[1], ct[2]};
  s.c = {c[0], c[1], c[2]};
  for (int i = 0; i < 9; ++i) { st.R[i] = Rt[i]; s.R[i] = R[i]; }
  double rad = P.dhat + P.bp_margin;
  build_anchors(P, S, st, broad_phase_state(P, st, rad));
  std::vector<Pair> C = broad_phase_state(P, s, rad);
  Grad G;
  double Ev = eval_energy(P, S, s, C, &G, parts);
  for (int v = 0; v < P.nv; ++v)
    for (int a = 0; a < 3; ++a) {
      g[3 * v + a] = G.g[v][a];
      for (int b = 0; b < 3; ++b) D[9 * v + 3 * a + b] = G.D[v][3 * a + b];
    }
  for (int a = 0; a < 3; ++a) { grig[a] = G.gc[a]; grig[3 + a] = G.gth[a]; }
  for (int i = 0; i < 9; ++i) { Drig[i] = G.Dc[i]; Drig[9 + i] = G.Dth[i]; }
  if (n_cand) *n_cand = C.size();
  if (n_anchor) *n_anchor = S.anchors.size();
  return Ev;
}
// p^T H p at (u, c, R) for direction (p, pc, pth); anchors at step start as in or_eval
double or_curvature(void* h, const double* u_t, const double* ct, const double* Rt, const double* u,
                    const double* c, const double* R, const double* p, const double* prig, const double* target7,
                    double dt) {
  Oracle* O = (Oracle*)h;
  Problem& P = O->P;
  Step S;
  S.cs = {target7[0], target7[1], target7[2]};
  S.Rs = quat_to_R(target7);
  S.h = dt;
  S.kappa = dt * dt * P.kappa_phys;
  S.eps = P.eps_v * dt;
  State st, s;
  st.u.resize(P.nv);
  s.u.resize(P.nv);
  std::vector<V3> pv(P.nv);
  for (int v = 0; v < P.nv; ++v) {
    st.u[v] = {u_t[3 * v], u_t[3 * v + 1], u_t[3 * v + 2]};
    s.u[v] = {u[3 * v], u[3 * v + 1], u[3 * v + 2]};
    pv[v] = P.fixed[v] ? V3{0, 0, 0} : V3{p[3 * v], p[3 * v + 1], p[3 * v + 2]};
  }
  st.c = {ct[0], ct[1], ct[2]};
  s.c = {c[0], c[1], c[2]};
  for (int i = 0; i < 9; ++i) { st.R[i] = Rt[i]; s.R[i] = R[i]; }
  double rad = P.dhat + P.bp_margin;
  build_anchors(P, S, st, broad_phase_state(P, st, rad));
  std::vector<Pair> C = broad_phase_state(P, s, rad);
  return curvature(P, S, s, C, pv, V3{prig[0], prig[1], prig[2]}, V3{prig[3], prig[4], prig[5]});
}
// One PNCG iteration's a6-a8 quantities at x_k = (u, c, R) of a step that started at
// (u_t, v_t, ct, Rt) with the given target: evaluation (O4b), |P g|_disp (O4d), the
// direction from the previous iterate's gradient / direction (O4e) and the step length
// (O4f, without the candidate-list cap of R16).  g_prev, p_prev: [nv*3 + 6] (gel, then c,
// theta).  out_p: [nv*3 + 6].  out[12]: beta, g^T p, g^T P g, restarted, M, alpha_upper,
// p^T H p, alpha_bar, alpha_ccd, alpha, L_rel, |P g|_disp.  (Test hook: kernel-level parity.)
void or_iteration(void* h, const double* u_t, const double* v_t, const double* ct, const double* Rt, const double* u,
                  const double* c, const double* R, const double* target7, double dt, const double* g_prev,
                  const double* p_prev, double gPg_prev, int restart, double* out_p, double* out) {
  Oracle* O = (Oracle*)h;
  Problem& P = O->P;
  Step S;
  S.h = dt;
  S.kappa = dt * dt * P.kappa_phys;
  S.eps = P.eps_v * dt;
  S.cs = {target7[0], target7[1], target7[2]};
  S.Rs = quat_to_R(target7);
  S.lam_t = O->eval_lam_t;
  S.lam_r = O->eval_lam_r;
  S.xhat_u.resize(P.nv);
  State st, s;
  st.u.resize(P.nv);
  s.u.resize(P.nv);
  Vecs gp, pp;
  gp.v.resize(P.nv);
  pp.v.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) {
    V3 a{u_t[3 * v], u_t[3 * v + 1], u_t[3 * v + 2]}, b{v_t[3 * v], v_t[3 * v + 1], v_t[3 * v + 2]};
    st.u[v] = a;
    S.xhat_u[v] = P.fixed[v] ? V3{0, 0, 0} : add(a, scl(dt, b));
    s.u[v] = {u[3 * v], u[3 * v + 1], u[3 * v + 2]};
    gp.v[v] = P.fixed[v] ? V3{0, 0, 0} : V3{g_prev[3 * v], g_prev[3 * v + 1], g_prev[3 * v + 2]};
    pp.v[v] = P.fixed[v] ? V3{0, 0, 0} : V3{p_prev[3 * v], p_prev[3 * v + 1], p_prev[3 * v + 2]};
  }
  const int o = 3 * P.nv;
  gp.c = {g_prev[o], g_prev[o + 1], g_prev[o + 2]};
  gp.th = {g_prev[o + 3], g_prev[o + 4], g_prev[o + 5]};
  pp.c = {p_prev[o], p_prev[o + 1], p_prev[o + 2]};
  pp.th = {p_prev[o + 3], p_prev[o + 4], p_prev[o + 5]};
  st.c = {ct[0], ct[1], ct[2]};
  s.c = {c[0], c[1], c[2]};
  for (int i = 0; i < 9; ++i) { st.R[i] = Rt[i]; s.R[i] = R[i]; }
  double rad = P.dhat + P.bp_margin;
  build_anchors(P, S, st, broad_phase_state(P, st, rad));
  std::vector<Pair> C = broad_phase_state(P, s, rad);
  Grad G;
  eval_energy(P, S, s, C, &G, nullptr);
  Vecs g = to_vecs(G);
  Vecs Pg = apply_P(P, G, g);
  double gPg = vdot(P, g, Pg);
  Direction Dn = direction(P, G, g, Pg, gPg, gp, pp, gPg_prev, restart != 0);
  StepLen SL = step_length(P, S, s, C, Dn.p, Dn.gp);
  for (int v = 0; v < P.nv; ++v)
    for (int a = 0; a < 3; ++a) out_p[3 * v + a] = Dn.p.v[v][a];
  for (int a = 0; a < 3; ++a) { out_p[o + a] = Dn.p.c[a]; out_p[o + 3 + a] = Dn.p.th[a]; }
  const double r[12] = {Dn.beta, Dn.gp, gPg, Dn.restarted ? 1.0 : 0.0, SL.M, SL.a_up, SL.q, SL.a_bar, SL.a_ccd,
                        SL.alpha, SL.Lrel, disp_norm(P, Pg)};
  for (int k = 0; k < 12; ++k) out[k] = r[k];
}
// alpha_ccd over the candidates at (u, c, R) for direction p (R15)
double or_alpha_ccd(void* h, const double* u, const double* c, const double* R, const double* p, const double* prig) {
  Oracle* O = (Oracle*)h;
  Problem& P = O->P;
  State s;
  s.u.resize(P.nv);
  Vecs pv;
  pv.v.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) {
    s.u[v] = {u[3 * v], u[3 * v + 1], u[3 * v + 2]};
    pv.v[v] = P.fixed[v] ? V3{0, 0, 0} : V3{p[3 * v], p[3 * v + 1], p[3 * v + 2]};
  }
  s.c = {c[0], c[1], c[2]};
  for (int i = 0; i < 9; ++i) s.R[i] = R[i];
  pv.c = {prig[0], prig[1], prig[2]};
  pv.th = {prig[3], prig[4], prig[5]};
  return alpha_ccd(P, s, broad_phase_state(P, s, P.dhat + P.bp_margin), pv);
}
// broad phase on explicit gel vertex coordinates in the indenter body frame gb [nv*3]
// out: (kind, a, b) triples; returns count (may exceed cap)
int or_broadphase_body(void* h, const double* gb, double r, int* out, int cap) {
  Problem& P = ((Oracle*)h)->P;
  std::vector<V3> g(P.nv);
  for (int v = 0; v < P.nv; ++v) g[v] = {gb[3 * v], gb[3 * v + 1], gb[3 * v + 2]};
  std::vector<Pair> C = broad_phase(P, g, r);
  for (size_t i = 0; i < C.size() && (int)i < cap; ++i) { out[3 * i] = C[i].kind; out[3 * i + 1] = C[i].a; out[3 * i + 2] = C[i].b; }
  return (int)C.size();
}
// broad phase at state (u, c, R), world coordinates formed as the oracle does
int or_broadphase_state(void* h, const double* u, const double* c, const double* R, double r, int* out, int cap) {
  Problem& P = ((Oracle*)h)->P;
  State s;
  s.u.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) s.u[v] = {u[3 * v], u[3 * v + 1], u[3 * v + 2]};
  s.c = {c[0], c[1], c[2]};
  for (int i = 0; i < 9; ++i) s.R[i] = R[i];
  std::vector<Pair> C = broad_phase_state(P, s, r);
  for (size_t i = 0; i < C.size() && (int)i < cap; ++i) { out[3 * i] = C[i].kind; out[3 * i + 1] = C[i].a; out[3 * i + 2] = C[i].b; }
  return (int)C.size();
}
// brute-force minimum distance over ALL primitive pairs at (u, c, R)
double or_dmin(void* h, const double* u, const double* c, const double* R) {
  Problem& P = ((Oracle*)h)->P;
  State s;
  s.u.resize(P.nv);
  for (int v = 0; v < P.nv; ++v) s.u[v] = {u[3 * v], u[3 * v + 1], u[3 * v + 2]};
  s.c = {c[0], c[1], c[2]};
  for (int i = 0; i < 9; ++i) s.R[i] = R[i];
  return brute_dmin(P, s);
}

// --- scalar pins ---
double or_barrier(double d, double dh, int deriv) {
  return deriv == 0 ? barrier_b(d, dh) : deriv == 1 ? barrier_db(d, dh) : barrier_ddb(d, dh);
}
double or_mollifier(double s, double eps, int deriv) { return deriv == 0 ? moll_f(s, eps) : moll_df(s, eps); }
double or_dist_pt(const double* p, const double* t0, const double* t1, const double* t2, double* w) {
  Dist D = dist_pt({p[0], p[1], p[2]}, {t0[0], t0[1], t0[2]}, {t1[0], t1[1], t1[2]}, {t2[0], t2[1], t2[2]});
  for (int k = 0; k < 4; ++k) w[k] = D.w[k];
  return D.d;
}
double or_dist_ee(const double* a0, const double* a1, const double* b0, const double* b1, double* w) {
  Dist D = dist_ee({a0[0], a0[1], a0[2]}, {a1[0], a1[1], a1[2]}, {b0[0], b0[1], b0[2]}, {b1[0], b1[1], b1[2]});
  for (int k = 0; k < 4; ++k) w[k] = D.w[k];
  return D.d;
}
// far-pair certificate of R15 on 4 corners z[12] (side A = first na corners): returns
// 1 if certified (separation >= dhat), g = the best separation found, n its plane normal
int or_certificate(const double* z12, int na, double dhat, double* g, double* n3) {
  V3 z[4];
  for (int k = 0; k < 4; ++k) z[k] = V3{z12[3 * k], z12[3 * k + 1], z12[3 * k + 2]};
  V3 n;
  bool ok = axis_separation(z, na, dhat, g, &n);
  for (int a = 0; a < 3; ++a) n3[a] = n[a];
  return ok ? 1 : 0;
}
double or_psi(double E, double nu, const double* F9) {
  Problem P;
  P.mu = E / (2 * (1 + nu));
  P.lam2 = E * nu / ((1 + nu) * (1 - 2 * nu)) + P.mu;
  M3 F;
  for (int i = 0; i < 9; ++i) F[i] = F9[i];
  return snh_psi(P, F);
}
void or_so3(const double* w, double* R, double* wlog) {  // exp and log round trip
  M3 Rm = so3_exp({w[0], w[1], w[2]});
  for (int i = 0; i < 9; ++i) R[i] = Rm[i];
  V3 l = so3_log(Rm);
  for (int i = 0; i < 3; ++i) wlog[i] = l[i];
}
void or_quat_to_R(const double* pose7, double* R) {
  M3 Rm = quat_to_R(pose7);
  for (int i = 0; i < 9; ++i) R[i] = Rm[i];
}

// The same NCG core on a quadratic E = 1/2 x^T A x - b^T x (pin of Eq. dk_direction + step_size):
// P = diag(A)^-1 (scalar) or identity, alpha = alpha_bar (alpha_upper -> inf).  Records iterates.
void or_ncg_quadratic(int n, const double* A, const double* b, const double* x0, int iters, int precond_identity,
                      int rule, double* xs) {
  std::vector<double> x(x0, x0 + n), g(n), gp(n), p(n), pp(n), Pg(n), y(n), Py(n);
  auto grad = [&](const std::vector<double>& xx, std::vector<double>& gg) {
    for (int i = 0; i < n; ++i) {
      double s = -b[i];
      for (int j = 0; j < n; ++j) s += A[i * n + j] * xx[j];
      gg[i] = s;
    }
  };
  auto Pm = [&](int i) { return precond_identity ? 1.0 : 1.0 / A[i * n + i]; };
  auto vd = [&](const std::vector<double>& a, const std::vector<double>& c) {
    double s = 0;
    for (int i = 0; i < n; ++i) s += a[i] * c[i];
    return s;
  };
  double gPg_prev = 1;
  for (int i = 0; i < n; ++i) xs[i] = x[i];
  for (int k = 0; k < iters; ++k) {
    grad(x, g);
    for (int i = 0; i < n; ++i) Pg[i] = Pm(i) * g[i];
    double gPg = vd(g, Pg);
    if (k == 0) for (int i = 0; i < n; ++i) p[i] = -Pg[i];
    else {
      for (int i = 0; i < n; ++i) { y[i] = g[i] - gp[i]; Py[i] = Pm(i) * y[i]; }
      double yp = vd(y, pp);
      double beta = ncg_beta(rule, vd(g, Py), yp, vd(y, Py), vd(pp, g), gPg, gPg_prev, vd(pp, pp));
      if (!std::isfinite(beta)) beta = 0;
      for (int i = 0; i < n; ++i) p[i] = -Pg[i] + beta * pp[i];
    }
    double gpv = vd(g, p);
    std::vector<double> Ap(n);
    for (int i = 0; i < n; ++i) { double s = 0; for (int j = 0; j < n; ++j) s += A[i * n + j] * p[j]; Ap[i] = s; }
    double a = std::min(step_alpha_upper(INF, 1.0), step_alpha_bar(gpv, vd(p, Ap)));
    if (!std::isfinite(a)) a = 0;
    for (int i = 0; i < n; ++i) x[i] += a * p[i];
    gp = g; pp = p; gPg_prev = gPg;
    for (int i = 0; i < n; ++i) xs[(k + 1) * n + i] = x[i];
  }
}

}  // extern "C"
