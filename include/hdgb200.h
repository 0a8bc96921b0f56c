/*
 * hdgb200.h - C ABI of the B200-native HDG trace-operator / multigrid hot path.
 *
 * Drop-in boundary for the reference `hdgmg` package (pure Python; its "plugin
 * API" is duck-typed).  Every entry point below replaces one
 * reference call site; a reference-side ctypes binding is in INTEGRATION.md.
 *
 * Conventions (all entry points):
 *   - plain C types only; vectors are fp64 DEVICE pointers in the reference's
 *     trace layout: block b of an interior facet holds n1 = p+1 contiguous values,
 *     blocks in `block_of` order (trace.py:39-41): interior horizontal facets row
 *     by row (j = 1..ny-1, i = 0..nx-1), then interior vertical facets column by
 *     column (i = 1..nx-1, j = 0..ny-1)  [mesh.py:112-117];
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *     all launches are asynchronous on it;
 *   - return 0 on success, nonzero on error; hdg_last_error() describes it
 *     (thread-local).  Inputs are never mutated (matvec_free / _cycle return new
 *     arrays in the reference).
 *   - ndof == 0 systems are legal (1x1 meshes) and every apply is a no-op
 *     (trace.py:90-91).
 */
#ifndef HDGB200_H
#define HDGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hdg_level hdg_level;       /* one trace operator on an nx x ny mesh at order p */
typedef struct hdg_transfer hdg_transfer; /* prolongation from level k+1 into level k */
typedef struct hdg_mg hdg_mg;             /* a level stack + workspaces + cached CUDA graphs */

enum { HDG_OK = 0, HDG_EINVAL = 1, HDG_ECUDA = 2, HDG_ENOMEM = 3, HDG_ESTATE = 4 };

const char* hdg_last_error(void);
int hdg_version(void);
/* number of kernel launches this thread issued through the library (for bench gpu_launches) */
int64_t hdg_launch_count(void);

/* ---------------------------------------------------------------- operators
 * Replaces TraceSystem's block state + matvec_free (trace.py:29-94) and
 * MGLevel.matvec / .operator (multigrid.py:204-207, 328-334).                  */

/* Shared-block operator (K = const, tau = const: SURVEY F2/F5): `block` is the
 * 4n1 x 4n1 row-major condensed block of an interior element (HOST pointer),
 * local slot = side*n1 + k, sides (bottom, right, top, left) [local.py:35-43]. */
int hdg_level_create_shared(int nx, int ny, int p, const double* block, hdg_level** out);

/* Stored-block operator: `blocks` is the reference `schur` stack (E, 4n1, 4n1)
 * row-major, element e = j*nx + i [trace.py:54], DEVICE pointer (caller keeps
 * ownership; it may be freed after the call).  Dirichlet columns must already
 * be zero (local.py:186-188); boundary-side rows are ignored. */
int hdg_level_create_stored(int nx, int ny, int p, const double* blocks, hdg_level** out);
/* The same stored operator filled by element-row chunks, for levels whose element blocks cannot
 * exist at once (configs[4]'s 8192^2 p=4 fine level: 214.7 GB of blocks, 107 GB of stream).
 * create_stored_empty allocates the stream; fill_stored_rows writes stream rows
 * [row0, row0 + nrows) from `blocks` = the element blocks of element rows
 * [max(row0 - 1, 0), row0 + nrows) (DEVICE, same layout as hdg_level_create_stored).  Every row
 * must be filled once before the level is applied. */
int hdg_level_create_stored_empty(int nx, int ny, int p, hdg_level** out);
int hdg_level_fill_stored_rows(hdg_level* lev, int row0, int nrows, const double* blocks, void* stream);
int hdg_level_destroy(hdg_level* lev);
int64_t hdg_level_ndof(const hdg_level* lev);
/* bytes the operator streams from HBM per apply (0 for shared: held in constant bank) */
int64_t hdg_level_operator_bytes(const hdg_level* lev);

/* Edge block-Jacobi smoother state (north star): D^-1 per
 * interior facet, D = that facet's diagonal n1 x n1 block of the operator.
 * Computed and inverted in-library from the level's own blocks. */
int hdg_level_set_blockjacobi(hdg_level* lev, double omega);

/* Chebyshev-weighted block-Jacobi: step k of m uses weight 1/theta_k, theta_k the Chebyshev
 * nodes of [lo, hi] (an interval of D^-1 A's spectrum; same rule as the reference FSAI sweep
 * weights, multigrid.py:76-81).  Needs hdg_level_set_blockjacobi first. */
int hdg_level_set_bj_chebyshev(hdg_level* lev, double lo, double hi);
/* `steps` (weighted) Jacobi sweeps in place; work: ndof scratch */
int hdg_bj_sweeps(const hdg_level* lev, const double* b, double* x, double* work, int steps,
                  void* stream);

/* y = A x  (trace.py:87-94) */
int hdg_matvec(const hdg_level* lev, const double* x, double* y, void* stream);

/* Facet-plane device layout (hdg_soa.cuh) for shared-block levels (constant coefficient on a
 * uniform mesh, p <= 8).  Replaces the same TraceSystem.matvec_free (trace.py:87-94) for callers
 * that keep their trace vectors resident on the device across many applies: node k of every
 * facet line is one contiguous run (boundary facets and pad slots stored as zeros), so the apply
 * streams coalesced rows with no shared-memory staging.
 *   hdg_soa_length  -> number of doubles of one facet-plane vector (prepares the level)
 *   hdg_soa_pack    -> reference layout (ndof) -> facet planes (writes every slot)
 *   hdg_soa_unpack  -> facet planes -> reference layout
 *   hdg_matvec_soa  -> y = A x in facet planes; writes every slot of y (not in place)
 * HDG_EINVAL for stored levels or an element block that is not mirror-invariant. */
int hdg_soa_length(hdg_level* lev, int64_t* n);
int hdg_soa_pack(hdg_level* lev, const double* x, double* x_soa, void* stream);
int hdg_soa_unpack(hdg_level* lev, const double* x_soa, double* x, void* stream);
int hdg_matvec_soa(hdg_level* lev, const double* x_soa, double* y_soa, void* stream);
/* r = b - A x; if norm2_out != NULL also writes ||b - A x||^2 (one double, device) */
int hdg_residual(const hdg_level* lev, const double* b, const double* x, double* r,
                 double* norm2_out, void* stream);
/* one damped block-Jacobi sweep x_out = x_in + omega D^-1 (b - A x_in); x_out != x_in */
int hdg_bj_sweep(const hdg_level* lev, const double* b, const double* x_in, double* x_out,
                 void* stream);

/* FSAI smoother (the reference default, multigrid.py:47-173): lower-triangular G and its
 * transpose in CSR (HOST arrays, int32 indices, sorted), lambda_max of G'GA, Chebyshev lower
 * fraction and omega.  Built on the host by the caller (fsai_build, multigrid.py:123-159). */
int hdg_level_set_fsai(hdg_level* lev, int64_t n, const int32_t* g_rowptr, const int32_t* g_cols,
                       const double* g_vals, int64_t nnz, const int32_t* gt_rowptr,
                       const int32_t* gt_cols, const double* gt_vals, double lam_max,
                       double cheb_fraction, double omega);
/* fsai_build's row solves (multigrid.py:133-152) on the device: for every row i of the
 * lower-triangular pattern (g_ptr/g_col, sorted, diagonal last; DEVICE arrays) solve
 * A[P_i, P_i] g = e_last by Cholesky and write g / sqrt(g_last) into g_val.  A in CSR on the
 * device (int32, sorted).  max_len >= the longest pattern row (<= 96).  *bad_row = the first
 * row whose principal block is not SPD (NotSPDError, multigrid.py:34), else -1.  Synchronises
 * the stream. */
int hdg_fsai_rows(int64_t n, const int32_t* a_ptr, const int32_t* a_col, const double* a_val,
                  const int32_t* g_ptr, const int32_t* g_col, double* g_val, int32_t max_len,
                  int64_t* bad_row, void* stream);
/* Facet-structured FSAI (hdg_fsai.cuh), the baseline pattern lower(A) of multigrid.py:127-131
 * built ON THE DEVICE from the level's element blocks: S_cls (C, 4n1, 4n1) DEVICE, elem_class
 * (E,) int64 DEVICE (element e = j nx + i -> class).  One Cholesky per facet gives its n1 rows of G
 * (multigrid.py:133-152); lambda_max(G'GA) by lam_iters power steps from the DEVICE start vector
 * v0 (the reference draws it with seed 1234, multigrid.py:162-173) -> *lam_max_out; Chebyshev
 * lower fraction and omega as FSAISmoother (multigrid.py:76-88).  A non-SPD principal system
 * returns HDG_ESTATE with *bad_row = the first failing DOF row (NotSPDError, multigrid.py:145-148).
 * p <= 8. */
int hdg_level_set_fsai_struct(hdg_level* lev, const double* S_cls, const int64_t* elem_class, const double* v0,
                              int lam_iters, double cheb_fraction, double omega, double* lam_max_out,
                              int64_t* bad_row, void* stream);
/* copy the structured factor to the host: gh (nx (ny-1) * n1 * 2n1), gv ((nx-1) ny * n1 * 6n1),
 * layout Gh[(k 2n1 + c) nh + f], Gv[(k 6n1 + c) nv + f] (hdg_fsai.cuh) */
int hdg_level_fsai_struct_get(const hdg_level* lev, double* gh, double* gv);
/* z = G'(G r)  (multigrid.py:72-74) */
int hdg_fsai_apply(const hdg_level* lev, const double* r, double* z, void* stream);
/* `steps` Chebyshev-weighted sweeps x <- x + w_k G'G(b - A x) in place (multigrid.py:83-88);
 * work_r, work_t: ndof scratch vectors */
int hdg_fsai_sweeps(const hdg_level* lev, const double* b, double* x, double* work_r,
                    double* work_t, int steps, void* stream);

/* ---------------------------------------------------------------- transfers
 * Replaces p_prolongation / h_prolongation (multigrid.py:215-298) as operators:
 * prolong_add: x_fine += P e_coarse;   restrict: r_coarse = P^T r_fine.        */

/* p-transfer on one mesh: V = n1f x (n1f-1) row-major (coarse GLL basis at fine GLL nodes) */
int hdg_transfer_create_p(const hdg_level* fine, const hdg_level* coarse, const double* V,
                          hdg_transfer** out);
/* h-transfer at p = 1 (n1 = 2): `halves` 2 x 2 x 2 (half index, fine node, coarse node);
 * `cross` = -V_f u_cols maps of the four cross facets (right of SW, right of NW, top of SW,
 * top of SE) of each coarse element: (ncross_sets, 4, 2, 8) row-major, HOST pointer;
 * ncross_sets = 1 (shared by every coarse element) or Ec = coarse element count. */
int hdg_transfer_create_h(const hdg_level* fine, const hdg_level* coarse, const double* halves,
                          const double* cross, int64_t ncross_sets, hdg_transfer** out);
/* the same on row WINDOWS of the meshes (multi-GPU strips): the fine level's mesh is rows
 * [fine_row0, fine_row0 + ny_fine) of the global fine mesh, the coarse level's rows
 * [coarse_row0, ...) of the global coarse mesh; cross maps are per WINDOW coarse element. */
int hdg_transfer_create_h_window(const hdg_level* fine, const hdg_level* coarse, const double* halves,
                                 const double* cross, int64_t ncross_sets, int fine_row0,
                                 int coarse_row0, hdg_transfer** out);
int hdg_transfer_destroy(hdg_transfer* t);
int hdg_prolong_add(const hdg_transfer* t, const double* e_coarse, double* x_fine, void* stream);
int hdg_restrict(const hdg_transfer* t, const double* r_fine, double* r_coarse, void* stream);

/* ---------------------------------------------------------------- multigrid
 * Replaces _cycle / v_cycle / w_cycle (multigrid.py:393-418) with a
 * device-resident cycle: level k's operator, BJ smoother and transfer k->k+1,
 * and a dense coarsest-level inverse (replaces splu, multigrid.py:209-212).    */
int hdg_mg_create(hdg_level* const* levels, hdg_transfer* const* transfers, int nlevels,
                  hdg_mg** out);
int hdg_mg_destroy(hdg_mg* mg);
/* coarsest-level inverse, n x n row-major HOST pointer, n = ndof of the last level */
int hdg_mg_set_coarse_inverse(hdg_mg* mg, const double* inv, int64_t n);
/* Cycle fusions (default on): (1) the trailing p = 1, block-Jacobi-smoothed, h-linked levels
 * whose top level has <= 2048 dofs run as ONE single-CTA shared-memory kernel; (2) on
 * constant-coefficient levels the first two Jacobi steps from x = 0 run as one trace kernel
 * (x1 = w1 D^-1 b formed on the staged tile).  Same recursion, buffers and weights as the
 * per-launch cycle (multigrid.py:393-406).  enable = 0 issues everything as separate launches
 * (A/B timing, parity tests). */
int hdg_mg_set_fused_tail(hdg_mg* mg, int enable);
/* Record-layout cycle: the constant-coefficient, block-Jacobi-smoothed p-ladder of the finest
 * mesh (levels 0 .. m-1, level m-1 is p = 1 and h-linked to level m) keeps every level vector as
 * facet records and runs each sweep / residual of multigrid.py:397-405 as one pass of the
 * record kernel with the update fused (first two sweeps from x = 0, residual + p-restriction,
 * p-prolongation + first post-sweep are single passes); b is packed and x unpacked at the
 * cycle's boundary, the levels below m use the reference layout.  mode 0: off, 1 (default):
 * when level 0 has p >= 2 and >= 2^13 dofs (env HDG_REC_MIN_DOF), 2: whenever the levels qualify, 3: as 2
 * with the p-prolongation as its own kernel, 4: as 2 with every qualifying h-coarsened level on
 * records too (automatically: those with >= 50k dofs, env HDG_REC_H_MIN_DOF; record-to-record
 * h-transfers).  hdg_mg_record_levels returns m of the last cycle (0: reference layout). */
int hdg_mg_set_records(hdg_mg* mg, int mode);
int hdg_mg_record_levels(const hdg_mg* mg);
/* hdg_mg_cycle on vectors that already live as facet records of level 0 (hdg_soa_pack): no
 * pack / unpack at the cycle's boundary; the last sweep writes x_rec directly.  Needs record
 * levels (HDG_ESTATE otherwise).  x0_rec may be NULL (zero guess) and may alias x_rec. */
int hdg_mg_cycle_records(hdg_mg* mg, const double* b_rec, const double* x0_rec, double* x_rec, int nu1,
                         int nu2, int visits, int use_graph, void* stream);
/* x = cycle(b, x0) with nu1/nu2 smoothing sweeps (FSAI if attached to the level, else
 * block-Jacobi), visits = 1 (V) or 2 (W).
 * x0 may be NULL (zero initial guess, as v_cycle(x0=None)).  x may alias x0.
 * If use_graph != 0 the launch sequence is captured once per (pointers, nu, visits)
 * into a CUDA graph and replayed. */
int hdg_mg_cycle(hdg_mg* mg, const double* b, const double* x0, double* x, int nu1, int nu2,
                 int visits, int use_graph, void* stream);
/* coarse solve on the last level alone: x = A_c^-1 b (multigrid.py:209-212) */
int hdg_coarse_solve(hdg_mg* mg, const double* b, double* x, void* stream);
/* CUDA graphs instantiated by hdg_mg_cycle so far (LRU cache of 8 per hierarchy; a smoother
 * change drops them all) */
int64_t hdg_mg_graph_captures(const hdg_mg* mg);

/* ---------------------------------------------------------------- solve loops
 * Replaces solve_mg (multigrid.py:421-439): cycles x <- cycle(b, x) until
 * ||b - A x|| <= tol ||b|| (checked before each cycle), at most max_cycles, stopping early when
 * the last 5 ratios are >= 1 (ConvergenceMonitor.diverged, multigrid.py:388-390).  x holds x0 on
 * entry and the iterate on return; res_hist (HOST, max_cycles + 1 doubles) receives
 * ||b - A x_k|| for k = 0..*ncycles.  One scalar D2H per cycle. */
int hdg_solve_mg(hdg_mg* mg, const double* b, double* x, int nu1, int nu2, int visits, double tol,
                 int max_cycles, double* res_hist, int* ncycles, void* stream);
/* Replaces TraceSystem.solve_cg (trace.py:142-163) with mg_preconditioner (multigrid.py:457-463):
 * conjugate gradients on `lev`, preconditioned by one V(nu1, nu2) cycle of `mg` from zero (mg may
 * be NULL: plain CG).  x0 = x if use_x0 else 0.  Stops when ||r|| <= tol ||b|| (checked at the top
 * of each iteration, as the reference) or after maxiter iterations; *iters = the reference's
 * returned count.  res_hist (HOST, maxiter + 1 doubles, may be NULL) receives ||r_k||.  The
 * iteration body is one CUDA graph; one scalar D2H per iteration. */
int hdg_pcg(const hdg_level* lev, hdg_mg* mg, const double* b, double* x, int use_x0, double tol, int maxiter,
            int nu1, int nu2, double* res_hist, int* iters, void* stream);

/* ---------------------------------------------------------------- reductions */
/* *out = sum_i a_i b_i (deterministic two-pass; device scalar out) */
int hdg_dot(const double* a, const double* b, int64_t n, double* out, void* stream);
/* CG vector updates (trace.py:156-161): x += alpha d, r -= alpha ad */
int hdg_cg_update(double* x, double* r, const double* d, const double* ad, double alpha, int64_t n,
                  void* stream);
/* d = z + beta d  (trace.py:161) */
int hdg_xpby(const double* z, double beta, double* d, int64_t n, void* stream);

/* ---------------------------------------------------------------- setup / post-solve kernels
 * the batched steps either side of the solve.  All pointers are
 * device pointers (fp64, row-major), one CTA per element unless noted.
 *
 * hdg_condense_piecewise: local.py:133-237 (local_blocks + assemble_local + condense) for an
 *   element-wise constant coefficient (isotropic or diagonal: kx, ky per element) and uniform tau,
 *   by eliminating the flux first: H = Stab + kx Lap0 + ky Lap1 (nb x nb, SPD) is eliminated on
 *   the augmented matrix [H | B], B = Tu - kx G0 - ky G1, in shared memory and
 *   S = kx A00 + ky A01 + Ms - B^T H^-1 B  (m = 4 (p+1), nb = (p+1)^2, S_out: E x m x m).
 *   *status (device int) is set to 1 on a non-positive pivot (NumericalBreakdown, local.py:27).
 * hdg_piecewise_usolve: rhs_e <- H(K_e)^-1 rhs_e in place (E x nb): the potential solve of
 *   condensed loads (local.py:236) and of the volume reconstruction (local.py:240-251).
 * hdg_gemm_nt: C = beta C + alpha diag(rowscale) ((A * colscale / adiv) B^T), A: E x J (lda), B: I x J,
 *   C: E x I (ldc); rowscale (E), colscale (J), adiv (E x J, ldad) may be NULL.  The shared-matrix
 *   products of reconstruct_all / postprocess_all (trace.py:171-185, local.py:282-299) and of the
 *   load condensation.
 * hdg_class_gemv: out_e = beta out_e + alpha M[cls_e] in_e with class-indexed I x J matrices
 *   (reconstruct_all with several element classes).
 * hdg_galerkin_p: S_c = Q^T S Q, Q = I_4 (x) V (multigrid.py:328-334 in element form);
 *   V: n1 x n1c.  hdg_galerkin_h: S_c = sum_k Q_k^T S_k Q_k over the 4 children at p = 1
 *   (S_children: C x 4 x 8 x 8; Q: C x 4 x 8 x 8, or one set when shared_q).
 * hdg_gather_elements: trace.py:81-85 for every element, lam_e: E x 4 (p+1), 0 on Dirichlet sides.
 * hdg_sum_owners: trace.py:67 / 73-79, rhs_f = cl[E1, side1] + cl[E2, side2] (slot-0 owner first). */
int hdg_condense_piecewise(int nb, int m, int64_t E, const double* kx, const double* ky, const double* stab,
                           const double* lap0, const double* lap1, const double* tu, const double* g0,
                           const double* g1, const double* a00, const double* a01, const double* ms,
                           double* S_out, int* status, void* stream);
int hdg_piecewise_usolve(int nb, int64_t E, const double* kx, const double* ky, const double* stab,
                         const double* lap0, const double* lap1, double* rhs, int* status, void* stream);
int hdg_gemm_nt(int64_t E, int I, int J, const double* A, int lda, const double* B, double* C, int ldc,
                const double* rowscale, const double* colscale, const double* adiv, int ldad, double alpha,
                double beta, void* stream);
int hdg_class_gemv(int64_t E, int I, int J, const int64_t* cls, const double* M, const double* in, int ldi,
                   double* out, int ldo, double alpha, double beta, void* stream);
int hdg_galerkin_p(int64_t E, int n1, int n1c, const double* S, const double* V, double* S_coarse, void* stream);
int hdg_galerkin_h(int64_t C, const double* S_children, const double* Q, int shared_q, double* S_coarse,
                   void* stream);
int hdg_gather_elements(int nx, int ny, int p, const double* lam, double* lam_e, void* stream);
int hdg_sum_owners(int nx, int ny, int p, const double* cl, double* rhs, void* stream);

/* ---------------------------------------------------------------- multi-GPU strips
 * element-row strips, one process (or context) per GPU.  Each rank holds a
 * WINDOW of the mesh (a level created on nx x nyl elements: its owned rows [r0, r1) of the global
 * mesh plus ghost rows, window row 0 = global row lo) and applies the single-GPU kernels to it;
 * hdg_dist_halo refreshes the ghost facet rows from the neighbouring ranks over the caller's NCCL
 * communicator (nccl_comm is an ncclComm_t; NCCL is resolved at run time from the process'
 * libnccl.so.2), packed / sent / received / unpacked on `stream` with no host wait:
 *   kind 0 (before an operator apply, trace.py:87-94 on the window): down: send h(r0), receive
 *          h(r0-1), v(r0-1); up: send h(r1-1), v(r1-1), receive h(r1);
 *   kind 1 (before an h-restriction, multigrid.py:276-281): send up v(r1-2), v(r1-1), h(r1-1).
 * (kind | 0x100: loopback self-test, the rank acts as its own lower and upper neighbour.)
 * hdg_dist_allreduce_sum: the owned-dof dot products / norms (one ncclAllReduce, in place). */
typedef struct hdg_dist hdg_dist;
int hdg_dist_init(void* nccl_comm, int rank, int nranks, hdg_dist** out);
int hdg_dist_destroy(hdg_dist* d);
int hdg_dist_halo(hdg_dist* d, const hdg_level* window_level, int lo, int r0, int r1, int ny_global, int kind,
                  double* x, void* stream);
int hdg_dist_allreduce_sum(hdg_dist* d, double* v, int count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HDGB200_H */
