// internal.h — device data layout and launchers of libtac (not part of the ABI).
//
// Layout (DESIGN.md §"Data layout in HBM"): per-env vectors are SoA with the env
// index fastest, A[c][v][Es] (Es = n_envs rounded up to 32), so a warp = 32 envs
// of one vertex / tet and every vertex row is one 128-byte coalesced transaction;
// the static mesh (tets, b-vectors, volumes, masses) is shared by all envs and
// read with warp-uniform broadcast loads.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tac {

constexpr int kNodeLeaf = 4;
constexpr int kRowSegMax = 16;  // cells per row segment at most (k_elem_grad_rows stages a segment's records per warp)
constexpr int kBvhW = 4;  // children per wide BVH node (8 measured slower: 1,430 vs 851 us per step-start broad phase, 120 registers)
constexpr int kBvhF4 = 3 * kBvhW / 2 + kBvhW / 4;  // float4 per wide node: boxes in pairs, refs four per float4
constexpr int kDedupSlots = 4096;  // per-env open-addressing table of shared constraints (R33)
// element tiles (k_elem_*_tiled): Morton-ordered tets grouped into tiles of <= kTileT tets
// touching <= kTileV vertices; each tile is scheduled into rounds of <= kTileW
// vertex-disjoint tets (one per warp) so shared-memory accumulation needs no atomics
constexpr int kTileT = 128, kTileV = 64, kTileW = 8;

struct BNode {  // indenter BVH node, body frame; leaf if left < 0: prims [-left-1, -left-1+right)
  float lo[3];
  int left;
  float hi[3];
  int right;
};

// friction anchor: frozen at the step start
// Delta_k(x) = sum_gel w u(x) + R Y_w + sig c - C0 with the indenter side folded into
// Y_w = sum_ind w Y (body frame), sig = sum_ind w, C0 = sum_gel w u^t + R^t Y_w + sig c^t
struct Anchor {  // friction anchor (R7): free gel corners carried by id, indenter side folded
  int gid[3];       // free gel corners: global vertex id, -1 if absent (fixed corners have u = 0)
  unsigned sid01;   // surface-local ids of gel corners 0 and 1 (16 bit each)
  float w[3], sig;  // weights of the gel corners; sig = sum of the indenter weights
  float t1[3], lam;
  float t2[3];
  unsigned sid2;    // surface-local id of gel corner 2
  float yw[3], pad2;  // Y_w = sum_ind w Y (body frame)
  double c0[3], pad3;  // C0 = sum_gel w u^t + R^t Y_w + sig c^t (Delta(x^t) = 0)
};

// per-env solver state (fp64 control, one thread per env in the scalar kernels)
struct EnvS {
  double c[3], R[9];          // current pose (trial point)
  double cp[3], Rp[9];        // pose at the last accepted iterate x_k
  double ct[3], Rt[9];        // pose at the step start
  double cs[3], Rs[9];        // target pose
  double gr[6], grp[6], pr[6];  // rigid gradient, previous gradient, direction (c, theta)
  double Dc[9], Dth[9];       // rigid diagonal blocks of the last accepted evaluation
  double E, Eprev, alpha, gp_prev, gPg_prev, S, beta, best_pg, pg, pose_res;
  double wt_acc, wr_acc;       // pose-spring weights psi'(r)/r at the last accepted point (k_alpha's curvature)
  double lam[6];               // pose multipliers (lam_t [N], lam_r [N m]) of the AL pose term (R29)
  double S2;                   // odometer of the pending candidate list since its build point (R16 pipeline)
  double cb[3], Rb[9];         // pose at the pending list's build point (the trial it is built at)
  int pending;                 // a candidate list is being rebuilt for this env (built during the
                               // evaluation after k_alpha listed it, activated by the vertex pre-pass after)
  int reb_iter;                // s.iter when it was listed
  double back;                 // u moves by back * p from the last evaluated point to the last accepted
                               // iterate x_k: 0 after an acceptance, -alpha of the rejected trial otherwise
                               // (a step that ends without converging commits x_k, never a trial)
  double Lrel_last;
  double odo, odo_base, Lc;   // classification odometer (R15 cache): path-length coordinate of the
                              // trial point / of x_k, L_rel of the current direction
  int cache_ok;               // candidate gap cache valid (same candidate list, classified once)
  int pad_cache;
  double Ep[5];                // energy parts of the last evaluation (diagnostics)
  double dbg[7];               // k_alpha's last p^T H p, M, L_rel, alpha_upper, alpha_bar, alpha_ccd, alpha
                               // before the candidate-list cap (diagnostics, tac_debug_iteration)
  int iter, halv, restart, reeval, mode, flags, best_it, accepted, rebuild, ncand_over;
  int ncand_max, nanc_last;   // per-step statistics (tac_env_stats)
};

// modes
constexpr int kActive = 0, kDone = 1;
// status flags (include/tac.h TAC_FLAG_*); a failed env is rolled back to x^t at finalize
constexpr int kFlagConv = 1, kFlagMaxIt = 2, kFlagNaN = 4, kFlagInfeas = 8, kFlagLarge = 16, kFlagOverflow = 32,
              kFlagStag = 64;
constexpr int kFlagFailed = kFlagNaN | kFlagInfeas | kFlagOverflow;

// double accumulators [kNAcc][Es]
enum AccIdx {
  A_EIN = 0, A_EEL, A_EB, A_EF,
  A_GR = 4,        // 6
  A_DR = 10,       // 18 (Dc 9, Dth 9)
  A_DOT = 28,      // 7: gPy, yp, yPy, pg, gPg, gg, pp
  A_PHP = 35,
  kNAcc = 36
};
// uint accumulators [kNAccU][Es] (non-negative floats compared as uint)
enum AccUIdx { U_PGMAX = 0, U_M, U_LREL, U_ACCD, U_GFAR, kNAccU };

struct Dev {
  // sizes
  int nv, nt, nsv, nse, nst, niv, nie, nit, nm, E, Es;
  int kmax, amax;
  // static mesh
  const int4* tets;      // [nt]
  const float4* tetb;    // [nt][3]: (b1, vol), (b2, fixed-corner mask bits), (b3, 0)
  const float4* X;       // [nv] rest position (fp32 exact), w = 0
  const float4* Xs;      // [nsv] rest positions of the gel-surface vertices (surface-local order)
  const float* mass;     // [nv]
  const float* smu;      // [nv] sum_e V_e mu |b_{e,v}|^2 (state-independent elastic diagonal / h^2)
  const unsigned char* vflag;  // [nv] bit0 fixed, bit1 on the gel surface
  const int* sv;         // [nsv]
  const int* svfree;     // [nsv] gel vertex id of a free surface vertex, -1 if fixed (near-pair scatter)
  const int2* se;        // [nse]
  const int4* st;        // [nst]
  const int2* se_l;      // [nse] surface-local vertex indices
  const int4* st_l;      // [nst] surface-local vertex indices
  int contact_bps;       // blocks per SM over the grid of the per-env contact passes (cgrid)
  int contact_smem;      // dynamic shared bytes of the staged contact kernels (0 = use the unstaged ones)
  cudaStream_t side, side2;  // per-simulator high-priority streams: the contact chain concurrent with the element pass
  cudaStream_t side3;        // the pipelined candidate rebuild (off the evaluation's critical path)
  cudaStream_t side4;        // the ind-gel point-triangle near pairs beside the gel-ind ones
  cudaEvent_t ev_fork, ev_join, ev_cls, ev_join2, ev_reb, ev_join4;
  const float4* Y;       // [niv] body frame, w = |Y|
  const int2* ie;        // [nie]
  const int4* it;        // [nit]
  const int* bvh_prims;  // prim lists
  const float4* bvh_pbox;  // [2 n_prims] per-prim box in leaf order: (lo, prim id bits), (hi, 0)
  int root_tri, root_edge, root_vert;  // binary-tree roots (host build; kernels start at the wide virtual roots)
  const float4* bvhw;    // [kBvhF4 n_wide] kBvhW-wide child-box nodes; wide nodes 0, 1, 2 = virtual roots (tri, edge, vert)
  const int4* mk_idx;    // [nm]
  const float4* mk_w;    // [nm]
  // per-env vectors [c][nv][Es]
  float *u, *ut, *vt, *uh, *g, *gp, *p, *D;
  float* Pg;             // [c][nv][Es] P g of the last direction reduction (k_dir_reduce -> k_dir_apply)
  float* Dcon;           // [nsv][Es/32][6][32] contact Gauss-Newton blocks of the surface vertices (barrier +
                         // friction), kept apart from D (elastic + inertia): a near-touching pair's block can
                         // exceed the elastic one by ~1e8, beyond fp32's precision in a sum; the block-Jacobi
                         // inverse forms D + Dcon in fp64 (R24)
  EnvS* es;              // [E]
  double* acc;           // [kNAcc][Es]
  unsigned* accu;        // [kNAccU][Es]
  float* dalpha;         // [Es] pending update u += dalpha p
  float* beta;           // [Es]
  int* run;              // [Es] bit0 evaluate, bit1 direction, bit2 rebuild
  float4* pcf;           // [Es] rigid p_c (float) for L_rel
  unsigned long long* cand;  // [2][E][kmax] (kind<<62 | a<<31 | b): two lists per env, lbuf[e] the active one,
                             // the other receives the pipelined in-loop rebuild (R16)
  uint2* ccorn;           // [2][E][kmax] corner ids of each candidate, 4 x 16 bit (gel: surface-local id,
                         // indenter: vertex id), written with the candidate list
  int* lbuf;             // [E] active candidate buffer (0 / 1)
  float* cgap;            // [E][kmax] certified axis gap + odometer at certification (rounded down)
  float4* cgeo;          // [E][kmax][2] near-pair geometry (d, n), (w0..w3) in near order: kinds 0, 1, 2 concatenated
  uint2* ncorn;          // [E][kmax] the near pairs' packed corner ids, same order as cgeo
  int* ncand;            // [2][E] candidates per buffer
  uint2* nearl;          // [E][3][kmax] packed corner ids of the near candidates (no far certificate), per pair kind
  int* nnear;            // [E][3]
  const int* sidx;       // [nv] surface-local index of a gel vertex, -1 if not on the surface
  float4* usurf;         // [nsv][Es] u of the surface vertices at the last evaluation
  float4* psurf;         // [nsv][Es] p of the surface vertices (current direction)
  Anchor* anc;           // [E][amax] (sorted per step by gel corners; see k_sort_anchors)
  Anchor* anc2;          // [E][amax] the other buffer of the per-step sort (pointers swapped)
  float* anc_f1;         // [E][amax] friction weight mu lambda f1(s) of the last evaluation
  int* nanc;             // [E]
  int* reb_list;         // [E] envs that rebuild their candidates in this iteration
  int* nreb;             // [1]
  // material / params
  float mu, lam2;        // mu, lambda' = lambda + mu of the create-time material (defaults)
  float* emat;           // [4][Es] per-env material: mu, lambda', mass scale rho_e / rho_0,
                         // elastic-diagonal scale mu_e / mu_0 (mass and sum V mu |b|^2 are stored for env 0's material)
  double* edbl;          // [2][Es] per-env kappa_phys, mu_f
  double noise_t, noise_r;  // per-step target pose noise amplitudes (R27; 0 = off)
  unsigned long long noise_seed;
  long long env_offset;  // global id of env 0 (sharded ranks draw the streams of their global envs)
  double rho_max, dhat, kappa_phys, eps_v, tol_x, k_t, k_r, f_max, t_max, ccd_s, bp_margin, c1, eps_E, mu_f;
  int beta_rule, precond, max_halv, stagnation, fixed_iters;
  int pose_al;           // augmented-Lagrangian pose enforcement (R29)
  int ee_moll;           // edge-edge parallel mollifier (R30)
  int dedup;             // IPC-toolkit constraint deduplication (R33)
  unsigned long long* dtab;  // [kDedupSlots][Es] claimed constraint keys of the current evaluation (R33)
  // element tiles
  int ntiles;
  const int* tile_vstart;        // [ntiles + 1] into tile_verts
  const int* tile_verts;         // global vertex ids
  const unsigned char* tile_vfl; // bit0 fixed, bit1 touched only by this tile
  const int* tile_tstart;        // [ntiles + 1] into tile_tv / tile_tb
  const uchar4* tile_tv;         // tile-local vertex indices of each tile tet
  const float4* tile_tb;         // [3 per tile tet] (b1, vol), (b2, 0), (b3, 0)
  const int* tile_rstart;        // [ntiles + 1] into tile_sched (in rounds)
  const short* tile_sched;       // [rounds][kTileW] tile-local tet index or -1
  // Kuhn cells (k_elem_grad_cells): 6 tets sharing a cell diagonal, corners relabelled to the
  // canonical pattern kCellTet; leftover tets go through the generic k_elem_grad
  int ncells, nrest;
  const int4* cell_v;            // [ncells][2] local corners 0-3, 4-7 (global vertex ids)
  const unsigned* cell_fix;      // [ncells] bit s: corner s fixed
  const float4* cell_tb;         // [ncells][6][3] (b1, vol), (b2, 0), (b3, 0) in canonical corner order
  const float4* cell_aa;         // [ncells] axis-aligned box (corner bit b along axis b): (1/s0, 1/s1, 1/s2, tet volume), else 0
  int cells_all_aa;              // every cell axis-aligned: the cell kernels compile the stored-B branch out
  const int2* cell_seg;          // [nseg] (first cell, count): runs of cells along corner bit 0 (cell order is chain order)
  int* alist;                    // [E] tolerance mode: envs evaluating next (run bit 0), built by k_alpha's last block
  int* glist;                    // [Es / 32] env groups holding one of them
  int* anum;                     // [2] sizes of alist / glist; -1: not built (identity mappings)
  unsigned* adone;               // k_alpha's block counter (last block builds the lists, resets it)
  // tolerance mode's WHILE graph body only: k_alpha's last block also runs the loop control
  // (continue while an env iterates and fewer than loop_limit trips ran): one launch less per trip
  int loop_on, loop_limit;
  int* loop_ctr;
  cudaGraphConditionalHandle loop_h;
  int remap_blocks;
  int compact;                   // tolerance mode: vertex / element passes over compacted env groups once the listed envs fill <= compact lanes per listed group on average (0: never)              // tolerance mode: CTAs dealt over the active envs' contact passes when few iterate
  int nseg, rows;                // rows: the gradient pass marches along the segments (all cells axis-aligned)
  const int* rest_tets;          // [nrest] tets not in any cell
  double t1[3], t2[3], nrm[3];
};

// ---- launchers (kernels.cu) ----
void launch_step_setup(const Dev& d, const float* poses, double h, unsigned long long step, cudaStream_t s);
void launch_vert_setup(const Dev& d, double h, cudaStream_t s);
void launch_broadphase(const Dev& d, bool masked, cudaStream_t s);
void launch_anchors(const Dev& d, double h, cudaStream_t s);
void launch_eval(const Dev& d, double h, cudaStream_t s);  // vertex pre + element + contact + accept
// apply = false: the convergence test and scalars only (the step's last evaluation: no new
// direction is needed, the step ends at the accepted iterate)
void launch_direction(const Dev& d, cudaStream_t s, bool apply = true);
void launch_curvature(const Dev& d, double h, cudaStream_t s);
void launch_alpha(const Dev& d, double h, cudaStream_t s);
void launch_finalize(const Dev& d, double h, cudaStream_t s);
void launch_intersect_check(const Dev& d, int* hit, cudaStream_t s);  // tac_create validation
void launch_sort_anchors(const Dev& d, Anchor* out, cudaStream_t s);  // per-step anchor order
void launch_markers(const Dev& d, float* out, int ncomp, cudaStream_t s);
void launch_marker_sqerr(const Dev& d, const float* ref, double* acc, int ncomp, cudaStream_t s);
void launch_reset(const Dev& d, const unsigned char* mask, const float* poses, cudaStream_t s);
void launch_status(const Dev& d, int* iters, float* pg, unsigned* flags, cudaStream_t s);
void launch_any_active(const Dev& d, int* out, cudaStream_t s);
void launch_loop_ctl(const Dev& d, cudaGraphConditionalHandle h, int* ctr, int limit, cudaStream_t s);
void launch_write_words(const Dev& d, uint64_t* dst, const uint64_t* words, int n, cudaStream_t s);  // n <= 8
void launch_stats(const Dev& d, int4* out, cudaStream_t s);
// debug
void launch_debug_broadphase(const Dev& d, double r, unsigned long long* out, int* cnt, int cap, cudaStream_t s);
void kernels_init(int contact_smem);  // per-device kernel attributes (call after cudaSetDevice)
int contact_smem_bytes(int nsv, int niv);  // 0 if the staged contact kernels do not fit
extern thread_local long long g_launches;

// ---- optional per-kernel CUDA-event profiling (bench.py roofline; off by default) ----
enum KernelId {
  KID_STEP_SETUP = 0, KID_VERT_SETUP, KID_BROADPHASE, KID_ANCHORS, KID_VERT_PRE, KID_ELEM_GRAD, KID_CONTACT_GRAD,
  KID_ACCEPT, KID_DIR_REDUCE, KID_DIR_SCALAR, KID_DIR_APPLY, KID_ELEM_CURV, KID_CONTACT_CURV, KID_ALPHA,
  KID_CCD, KID_FIN_VERT, KID_FIN_ENV, KID_MARKERS, KID_OTHER, KID_CONTACT_CLASSIFY,
  KID_CONTACT_NEAR_IG, KID_CONTACT_NEAR_EE, KID_CONTACT_FRICTION, KID_BROADPHASE_LIST, KID_DIR_REDUCE_SURF,
  KID_COUNT
};
struct Profiler;
extern thread_local Profiler* g_prof;
void prof_begin(int kid, cudaStream_t s);
void prof_end(int kid, cudaStream_t s);
const char* kernel_name(int kid);
// optional per-stream timeline of one iteration (TAC_TIMELINE=1; measurement only): an event
// recorded on the launching stream after every launch, streams kept concurrent
extern thread_local bool g_tl_on;
void tl_mark(int kid, cudaStream_t s);

}  // namespace tac
