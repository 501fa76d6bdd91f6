/* tac.h — C ABI of the B200-native batched PNCG-IPC tactile stepper.
 *
 * The library (paper_2603_28475_b200/libtac.so) runs the data-parallel hot path of
 * Tac2Real (arXiv 2603.28475) for n_envs independent environments on one GPU:
 * one implicit-Euler time step of a tetrahedral gel pad pressed by a rigid
 * indenter, minimising the incremental potential of Supp. Eq. (ipc_energy)
 * with the preconditioned Dai-Kou nonlinear CG of
 * Eq. (dk_direction) and the step bound of Eq. (step_size)
 * (P:459-463), followed by the marker displacement field.
 * Readings where the paper is silent are numbered R# in DESIGN.md.
 *
 * Conventions shared by every call
 *   - Units: SI (m, kg, s).  Gel frame: +z is the outward normal of the contact face.
 *   - Pose: 7 floats (t_x, t_y, t_z, q_w, q_x, q_y, q_z) mapping the indenter body
 *     frame into the gel frame.  The quaternion is normalised in fp64 internally.
 *   - Host pointers are read during the call only (deep copies are taken).
 *   - Device pointers are caller-owned (e.g. torch tensors' data_ptr()); they are
 *     read / written asynchronously on the caller's `stream` (a cudaStream_t passed
 *     as void*; NULL = legacy default stream), so the caller keeps them alive until
 *     the stream has passed the call.
 *   - Every call returns a tac_status.  A failing call leaves a message retrievable
 *     with tac_last_error().  CUDA errors are sticky (TAC_ECUDA) until tac_destroy.
 *   - A handle is bound to one device and is not thread-safe; distinct handles may
 *     run concurrently (one handle per GPU).
 *   - A per-environment solver failure is NOT a call failure: it sets a bit in the
 *     env's flags (TAC_FLAG_*) and rolls that env back to its step-start state.
 */
#ifndef TAC_H_
#define TAC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t tac_status;
#define TAC_OK 0
#define TAC_EINVAL 2   /* invalid input (mesh, parameters, pointers, sizes) */
#define TAC_ESOLVER 3  /* reserved: whole-call solver failure */
#define TAC_ECUDA 4    /* CUDA runtime error (sticky) */
#define TAC_ENOMEM 5   /* device allocation failed */
#define TAC_ESTATE 6   /* call not valid in the handle's state */

/* per-env status flags (tac_env_status) */
#define TAC_FLAG_CONVERGED 1u   /* |P g|_disp <= tol_x (tolerance mode) */
#define TAC_FLAG_MAXITER 2u     /* iteration budget used (always set in fixed-iteration mode) */
#define TAC_FLAG_NAN 4u         /* non-finite energy at the step start: env rolled back */
#define TAC_FLAG_INFEASIBLE 8u  /* a candidate pair reached d <= 0 at the step start: rolled back */
#define TAC_FLAG_LARGE_MOTION 16u /* target pose > 2 mm or > 5 deg from the current pose */
#define TAC_FLAG_OVERFLOW 32u   /* candidate or anchor capacity exceeded: pairs would be dropped, so the
                                  step fails at its next evaluation and the env is rolled back */
#define TAC_FLAG_STAGNATION 64u /* no decrease of |P g|_disp over `stagnation` iterations */

/* Gel tetrahedral mesh (Supp. §A "We discretize the sensor gel using a tetrahedral
 * mesh").  rest_xyz [n_verts][3] metres; tets [n_tets][4] with positive
 * orientation det[x1-x0, x2-x0, x3-x0] > 0; fixed [n_fixed] = Dirichlet (bonded base). */
typedef struct {
  int32_t n_verts;
  const double* rest_xyz;
  int32_t n_tets;
  const int32_t* tets;
  int32_t n_fixed;
  const int32_t* fixed;
} tac_tet_mesh;

/* Rigid indenter: closed triangle shell in its body frame (metres). */
typedef struct {
  int32_t n_verts;
  const double* rest_xyz;
  int32_t n_tris;
  const int32_t* tris;
} tac_tri_mesh;

/* Stable Neo-Hookean material (DESIGN R1) + Coulomb friction coefficient:
 * E [Pa], nu [-], rho [kg/m^3], mu_f [-]  (theta = [E, nu, rho, mu] of Sec. 4.2). */
typedef struct {
  double E, nu, rho, mu_f;
} tac_material;

/* Markers: rest positions [rows*cols][3] on the contact face, row-major;
 * output frame t1, t2 (tangent), n (normal).  mode 0 = barycentric weights of the
 * enclosing rest tet (default, R22); mode 1 = k nearest gel surface vertices with
 * inverse-distance weights (1 <= k <= 4). */
typedef struct {
  int32_t rows, cols;
  const double* rest_xyz;
  double t1[3], t2[3], n[3];
  int32_t mode, k;
} tac_marker_set;

/* Solver parameters (defaults in DESIGN.md Appendix "constants"):
 *   dhat [m]        barrier activation distance d^
 *   kappa_phys [N/m] barrier stiffness; the objective uses kappa = dt^2 kappa_phys (R4);
 *                   <= 0 selects the default rule 0.2 E lbar^2 / (12.25 dhat)
 *   eps_v [m/s]     friction velocity threshold, eps = eps_v dt
 *   tol_x [m]       convergence on |P g|_disp (R17); tolerance mode only
 *   k_t [N/m], k_r [N m/rad], f_max [N], t_max [N m]   force-capped pose spring (R18)
 *   ccd_s           conservative-advancement fraction s (R15)
 *   bp_margin [m]   candidate margin m_r; candidates within r = dhat + m_r (R16)
 *   c1, eps_E       Armijo constant and relative energy noise allowance (R14)
 *   max_iters       iteration budget per step (tolerance mode)
 *   fixed_iters     > 0: run exactly this many iterations per step (benchmark mode).
 *                   A step that ends without converging (fixed mode, or max_iters reached)
 *                   commits its last ACCEPTED iterate, never an unevaluated or rejected trial
 *                   (R31); the budget's last evaluation computes no new direction.
 *   beta_rule       0 Dai-Kou, 1 PR+, 2 FR, 3 DK+ (max(beta_DK, 0.5 g^T p/|p|^2), R28);
 *                   outside 0..3 -> TAC_EINVAL
 *   precond         0 3x3 block Jacobi, 1 scalar Jacobi P = diag(H)^-1; else TAC_EINVAL
 *   max_halvings    Armijo halvings before restarting along -P g
 *   stagnation      iterations without |P g| progress before giving up (0 = off)
 *   max_candidates  per-env capacity of candidate pairs (0 = default 32768; an env that
 *                   exceeds it fails its step, TAC_FLAG_OVERFLOW)
 *   max_anchors     per-env capacity of friction anchors (0 = default 4096; at most 16384)
 *   check_every     tolerance mode: host polls "all envs done" every N iterations
 *   pose_al         1: augmented-Lagrangian pose enforcement (R29): the pose
 *                   term gains h^2 (lam_t . (c - c*) + lam_r . log(R R*^T)) with per-env multipliers,
 *                   updated after every step by the spring force, lam += psi'(r) r/|r| (reset by
 *                   tac_reset); 0: plain penalty (default).  Outside {0, 1} -> TAC_EINVAL
 *   ee_mollifier    1: IPC's edge-edge mollifier (R30): an edge-edge pair's
 *                   barrier becomes m(c) kappa b(d), c = |e_a x e_b|^2, m = -c^2/eps^2 + 2c/eps below
 *                   eps = 1e-3 |E_a|^2 |E_b|^2 (rest lengths), 1 above; its friction lambda too.
 *                   0: off (default).  Outside {0, 1} -> TAC_EINVAL
 *   dedup           1: IPC-toolkit constraint deduplication (R33): a pair's
 *                   constraint is its closest features (corners with a non-zero closest-point
 *                   weight); point-edge and point-point constraints, realised by several
 *                   point-triangle / edge-edge pairs, carry their barrier and friction anchor once
 *                   (the mollifier then applies to edge-edge constraints only).  0: the literal sum
 *                   over pairs of P:432 (default).  Outside {0, 1} -> TAC_EINVAL */
typedef struct {
  double dhat, kappa_phys, eps_v, tol_x, k_t, k_r, f_max, t_max, ccd_s, bp_margin, c1, eps_E;
  int32_t max_iters, fixed_iters, beta_rule, precond, max_halvings, stagnation;
  int32_t max_candidates, max_anchors, check_every, pose_al, ee_mollifier, dedup;
} tac_solver_params;

typedef struct {
  const tac_tet_mesh* gel;
  const tac_material* mat;
  const tac_marker_set* markers;
  const tac_tri_mesh* indenter;
  const tac_solver_params* params;
  int32_t n_envs;
  int32_t device;            /* CUDA device ordinal */
  const float* init_poses;   /* host [n_envs][7] initial indenter poses */
} tac_create_info;

typedef struct tac_sim tac_sim; /* opaque, owned by the library */

/* Validate inputs, precompute (rest shape, lumped masses, gel surface, indenter BVHs,
 * fp64 marker location), allocate all device state and set every env to rest with
 * its initial pose.  Errors: TAC_EINVAL (non-positive tet volume, index out of range,
 * marker outside the mesh, indenter touching the gel at its initial pose, bad
 * parameters), TAC_ENOMEM, TAC_ECUDA.  On error *out is NULL. */
tac_status tac_create(const tac_create_info* info, tac_sim** out);

/* One implicit-Euler step of all envs to the target indenter poses
 * target_poses (device, [n_envs][7] fp32) with time step dt > 0.
 * setup, broad phase, friction anchors, the PNCG-IPC loop,
 * finalize.  Asynchronous on `stream`. */
tac_status tac_step(tac_sim* sim, const float* target_poses, float dt, void* stream);

/* Marker displacement field (row a10): out (device, [n_envs][rows*cols][ncomp] fp32)
 * = (u_m.t1, u_m.t2[, u_m.n]) with u_m = sum_j w_mj u_j.  ncomp in {2, 3}. */
tac_status tac_markers(tac_sim* sim, float* out, int32_t ncomp, void* stream);

/* ---- marker all-gather to the policy rank (SURVEY §8b "L4", §8e; one
 * set of environments per GPU, the marker fields go to the policy) ----
 * NCCL is resolved at run time (dlopen of the libnccl.so.2 the process already loaded, e.g.
 * torch's, else the system one): libtac.so itself has no NCCL dependency.  TAC_EINVAL if NCCL
 * cannot be loaded.
 *
 * tac_nccl_unique_id: out = a fresh 128-byte ncclUniqueId (call on one rank, share the bytes
 *   with the others out of band, e.g. a torch.distributed broadcast).
 * tac_nccl_comm_create: ncclCommInitRank(nranks, id, rank) on CUDA device `device`; *comm is
 *   an opaque ncclComm_t owned by the caller (collective call: every rank must enter it).
 * tac_nccl_comm_destroy: ncclCommDestroy.
 * tac_gather_markers: writes this simulator's marker field ([n_envs][rows*cols][ncomp], as
 *   tac_markers) into slot `rank` of recvbuf (device fp32 [nranks * n_envs][rows*cols][ncomp],
 *   rank = the comm's rank) and all-gathers the slots in place on `stream` (ncclAllGather,
 *   NVLink / NVSwitch between the GPUs of a node).  Every rank must hold the same n_envs and
 *   ncomp.  Asynchronous on `stream`; TAC_EINVAL on a null pointer or bad ncomp, TAC_ECUDA
 *   on an NCCL failure (message in tac_last_error). */
tac_status tac_nccl_unique_id(uint8_t out[128]);
tac_status tac_nccl_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, void** comm);
tac_status tac_nccl_comm_destroy(void* comm);
tac_status tac_gather_markers(tac_sim* sim, void* nccl_comm, float* recvbuf, int32_t ncomp, void* stream);

/* Per-step target pose noise (PAPER.md Table "Parameters Randomization Range", P:693-694,
 * "IPC Rand. Move. Noise", and P:726 "a small random movement on holding object" at each
 * timestep; reading DESIGN.md R27).  From the next tac_step on, env e's target
 * at step k (k = number of tac_step calls since create) is c_s += sigma_t (u0, u1, u2) [m],
 * R_s <- exp([sigma_r (u3, u4, u5)]) R_s [rad], u uniform on (-1, 1) from Philox4x32-10 with
 * key = seed and counter = (env_offset + e, k_lo, k_hi, 0 / 1).  sigma_t = sigma_r = 0 turns
 * it off (the default).  env_offset >= 0 is this simulator's first global env id (sharded
 * ranks reproduce a single-process run).  TAC_EINVAL on negative arguments. */
tac_status tac_set_pose_noise(tac_sim* sim, double sigma_t, double sigma_r, uint64_t seed, int64_t env_offset);

/* Calibration loss term (Eq. 6, L = 1/(K N) sum_k sum_i |u_sim - u_real|^2):
 * acc[e] += sum over markers and the ncomp components of (u_m(theta_e) - ref[e][m])^2,
 * u_m computed exactly as tac_markers does.  ref: device fp32 [n_envs][rows*cols][ncomp];
 * acc: device fp64 [n_envs], accumulated (zero it once per trajectory).  ncomp in {2, 3}.
 * Asynchronous on `stream`. */
tac_status tac_marker_sqerr(tac_sim* sim, const float* ref, double* acc, int32_t ncomp, void* stream);

/* Checkpoint / resume: the state one step carries into the next -- u^t, v^t
 * of every env, the per-env pose / multipliers / statistics record and the step counter that
 * keys the pose-noise streams (R27).  Candidate lists and anchors are rebuilt at every step
 * start, so they are not part of it.  `bytes` receives the size of a checkpoint; `dst` /
 * `src` are caller-owned DEVICE buffers of at least that size on the handle's device.
 * Save is asynchronous on `stream`; load validates the buffer's header (TAC_EINVAL if it was
 * written by a simulator of another size) and therefore synchronises `stream` once before
 * its asynchronous device-to-device copies.  Loading a checkpoint and stepping with the
 * same targets reproduces the steps taken after the save (up to the order of fp32 atomic
 * sums). */
tac_status tac_checkpoint_size(const tac_sim* sim, uint64_t* bytes);
tac_status tac_checkpoint_save(tac_sim* sim, void* dst, void* stream);
tac_status tac_checkpoint_load(tac_sim* sim, const void* src, void* stream);

/* Re-initialise the envs with env_mask[e] != 0 (device uint8 [n_envs]) to rest,
 * zero velocity and pose poses[e] (device fp32 [n_envs][7]). */
tac_status tac_reset(tac_sim* sim, const uint8_t* env_mask, const float* poses, void* stream);

/* Per-env material theta_e = [E, nu, rho, mu_f] (PAPER.md Sec. "material calibration",
 * Eqs. 6-7: the calibration searches theta over a batch of environments;
 * SURVEY §8f-2).  Each pointer is a HOST array of n_envs doubles, or NULL to keep that
 * parameter; E > 0, 0 <= nu < 0.5, rho > 0, mu_f >= 0 per env, else TAC_EINVAL and
 * nothing changes.  Takes effect at the next tac_step: Lame parameters (SNH),
 * lumped masses, the elastic diagonal blocks, the friction coefficient and,
 * with the default kappa rule (kappa_phys == 0 at create, R4), the barrier stiffness
 * 0.2 E lbar^2 / (12.25 dhat).  The upload is ordered on `stream` after the work already
 * queued there (a tac_step in flight on it finishes with the old tables) and the call returns
 * once it has landed (it synchronises `stream`). */
tac_status tac_set_env_material(tac_sim* sim, const double* E, const double* nu, const double* rho,
                                const double* mu_f, void* stream);

/* Per-env diagnostics of the last step (device outputs [n_envs], any may be NULL):
 * iterations used, |P g|_disp at exit, flags (TAC_FLAG_*). */
tac_status tac_env_status(tac_sim* sim, int32_t* iters, float* pg_norm, uint32_t* flags, void* stream);

/* Per-env statistics of the last step (device int32 [n_envs][4]): iterations,
 * peak candidate-pair count, friction anchors, candidate rebuilds inside the loop. */
tac_status tac_env_stats(tac_sim* sim, int32_t* out, void* stream);

/* Sizes: out[0..9] = n_verts, n_tets, n_envs, env_stride, n_markers, n_surface_verts,
 * n_surface_edges, n_surface_tris, n_kuhn_cells (6 tets each, register-blocked gradient),
 * n_other_tets (generic gradient). */
tac_status tac_info(const tac_sim* sim, int32_t* out);

/* Number of kernel launches issued by the last tac_step / tac_markers call.  In tolerance
 * mode the iteration loop runs under device-side control (a CUDA-graph WHILE node); its trip
 * count is then read back from the device, so this call synchronises the device. */
int64_t tac_last_launch_count(const tac_sim* sim);

/* Per-kernel timing (profiling hook used by bench.py for the roofline): when enabled,
 * every kernel launched by tac_step / tac_markers is bracketed by CUDA events recorded
 * on the launching stream.  tac_profile_read synchronises, returns for the first n
 * kernel ids (see tac_profile_kernel_name) the summed milliseconds and launch counts
 * since the last read, and resets them.  TAC_ESTATE if profiling is off. */
tac_status tac_profile_enable(tac_sim* sim, int32_t on);
tac_status tac_profile_read(tac_sim* sim, double* ms, int64_t* counts, int32_t n);
const char* tac_profile_kernel_name(int32_t id); /* NULL-safe; "?" beyond the last id */

tac_status tac_destroy(tac_sim* sim);

/* Message of the last failing call on this handle (or of the last failed tac_create
 * when sim is NULL).  Owned by the library. */
const char* tac_last_error(const tac_sim* sim);

/* ---- test / debug hooks (synchronous, host buffers, one env at a time) ---- */

/* Host copies of env state: u, v [n_verts][3] (displacement from rest, velocity),
 * c [3], R [9] row-major (current step-start pose). */
tac_status tac_get_state(tac_sim* sim, int32_t env, double* u, double* v, double* c, double* R);
tac_status tac_set_state(tac_sim* sim, int32_t env, const double* u, const double* v, const double* c,
                         const double* R);

/* Candidate set of env `env` at state (u fp32 [n_verts][3], c, R fp64) with radius r,
 * computed by the device broad phase.  out [cap][3] = (kind, a, b): kind 0 = (gel
 * surface vertex a, indenter tri b), 1 = (indenter vertex a, gel surface tri b),
 * 2 = (gel surface edge a, indenter edge b); surface primitives are numbered as
 * tac_debug_surface returns them.  *n = number found (may exceed cap). */
tac_status tac_debug_broadphase(tac_sim* sim, int32_t env, const float* u, const double* c, const double* R,
                                double r, int32_t* out, int32_t cap, int32_t* n);

/* Gel surface primitives: sv [n_sv], se [n_se][2], st [n_st][3]; indenter edges ie [n_ie][2]
 * (sizes from tac_info and counts[0] = n_ie). */
tac_status tac_debug_surface(const tac_sim* sim, int32_t* sv, int32_t* se, int32_t* st, int32_t* ie,
                             int32_t* counts);

/* Marker map computed at create: tet [M], idx [M][4], w [M][4] (fp64 weights). */
tac_status tac_debug_marker_map(const tac_sim* sim, int32_t* tet, int32_t* idx, double* w);

/* Energy parts [5] (inertia, elastic, barrier, friction, pose), gradient g [n_verts][3],
 * diagonal blocks D [n_verts][9], rigid gradient grig [6] = (g_c, g_theta) and rigid
 * blocks Drig [18] of env `env` at state (u, c, R) with friction anchors built at the
 * step-start state (u_t, v_t, c_t, R_t), target pose target7 and step dt; the same
 * kernels as tac_step.  Overwrites the env's state. */
tac_status tac_debug_eval(tac_sim* sim, int32_t env, const double* u_t, const double* v_t, const double* c_t,
                          const double* R_t, const double* u, const double* c, const double* R,
                          const double* target7, double dt, double* parts, double* g, double* D, double* grig,
                          double* Drig);

/* One PNCG iteration's a6-a8 quantities (SURVEY §4 tier 2, kernel-level parity of the
 * direction, curvature and step bounds): as tac_debug_eval at x_k = (u, c, R), then the
 * direction from the previous iterate's gradient g_prev and direction p_prev ([n_verts*3 + 6]
 * each: gel, then c, theta; fixed vertices ignored), gPg_prev = g_prev^T P_prev g_prev (used
 * by the PR+ / FR rules) and restart != 0 (p = -P g), then the curvature and step-length
 * kernels.  p_out [n_verts*3 + 6] = the new direction; out[12] = beta, g^T p, g^T P g,
 * restarted (beta == 0), M = |p|_disp, alpha_upper, p^T H p, alpha_bar
 * (P:461), alpha_ccd (R15), alpha (before the candidate-list cap of R16), L_rel,
 * |P g|_disp.  Same kernels as tac_step; overwrites the env's state. */
tac_status tac_debug_iteration(tac_sim* sim, int32_t env, const double* u_t, const double* v_t, const double* c_t,
                               const double* R_t, const double* u, const double* c, const double* R,
                               const double* target7, double dt, const double* g_prev, const double* p_prev,
                               double gPg_prev, int32_t restart, double* p_out, double* out);

#ifdef __cplusplus
}
#endif
#endif /* TAC_H_ */
