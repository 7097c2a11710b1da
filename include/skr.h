/* skr.h -- C ABI of the B200-native SKR hot path (libskr.so).
 *
 * Plain pointers, sizes and a cudaStream_t passed as void*; no torch types.
 * All device pointers must be device-resident (cudaMalloc / torch CUDA tensors).
 * Compute entry points allocate no device memory: the caller passes a
 * workspace sized by the *_workspace_bytes() query. Every entry point returns
 * an int status (SKR_OK = 0); no C++ exception crosses the ABI.
 *
 * Reference interfaces replaced (kryrec v0.1.0, /root/reference/pkg/src/kryrec):
 *   skr_spmv            <- sparse.spmv (sparse.py:155-160) and the operator of
 *                          gmres.make_operator (gmres.py:184-190) with
 *                          JacobiPreconditioner.apply (precond.py:66-77)
 *   skr_gcrodr_solve    <- gcrodr.gcrodr_solve (gcrodr.py:295-496), including
 *                          refresh_recycle (gcrodr.py:80-113) and the recycle
 *                          update (gcrodr.py:444-460); k == 0 is the
 *                          gmres_solve path (gmres.py:193-267, gcrodr.py:326-330)
 *   skr_sort_dist2 /
 *   skr_sort_chain      <- sorting.greedy_sort / _greedy_chain (sorting.py:55-80)
 *   skr_dense_hr_first  <- gcrodr.harmonic_ritz_first_cycle (gcrodr.py:173-206)
 *   skr_dense_hr_next   <- gcrodr.harmonic_ritz_subsequent (gcrodr.py:209-240)
 *   skr_precond_build /
 *   skr_precond_apply   <- precond.build_preconditioner (precond.py:251-312) and
 *                          the SOR / ILU(0) / IC(0) / block-Jacobi apply
 *                          (precond.py:80-145)
 */
#ifndef SKR_H_
#define SKR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum skr_status_code {
  SKR_OK = 0,
  SKR_ERR_ARG = 1,          /* bad argument (ValueError in the reference) */
  SKR_ERR_WORKSPACE = 2,    /* workspace too small */
  SKR_ERR_CUDA = 3,         /* CUDA runtime error */
  SKR_ERR_TIMEOUT = 4,      /* device barrier / host wait timed out */
  SKR_ERR_UNSUPPORTED = 5,  /* configuration beyond compiled limits */
};

/* CSR matrix, int32 indices, fp64 values, device pointers. diag == NULL means
 * no preconditioner (IdentityPreconditioner); otherwise the Jacobi diagonal
 * (the left preconditioner M = diag(A), applied as an IEEE division). */
typedef struct skr_csr {
  int32_t n;
  int32_t nnz;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* values;
  const double* diag;
  /* Optional symmetric 7-diagonal form of the same matrix (NULL = none),
   * built by skr_stencil_build with diagonal offsets sx (and sxy, 0 in 2-D).
   * Every kernel applying A uses it when the build verified that the CSR
   * qualifies (results bit-identical to the CSR row sums), else the CSR. */
  const void* stencil;
  int32_t sx;
  int32_t sxy;
  /* Optional general left preconditioner (NULL = none): a device buffer built
   * by skr_precond_build from this matrix (SOR, ILU(0), IC(0), block Jacobi).
   * When set it replaces diag: every op(v) = M^-1 (A v) and every
   * preconditioned residual solves M z = v with the stored factorization. */
  const void* precond;
  int32_t precond_kind; /* skr_precond_kind of `precond` (0: read from the buffer) */
} skr_csr;

/* SolverConfig (gmres.py:26-43) + one launch knob. */
typedef struct skr_config {
  int32_t m;
  int32_t k;
  int32_t max_iter;
  int32_t grid_ctas; /* CTAs of the persistent Arnoldi kernel; 0 = fill the GPU.
                        Callers running several chains concurrently on one GPU
                        give each chain a share (e.g. 2 * SMs / chains * 2). */
  double tol;
  int32_t flags;     /* SKR_COLLECT_DIAGNOSTICS: log (stage, k, ||op U - C||_F,
                        ||C^T C - I||_F) after the refresh and after every deflated
                        cycle's recycle update, read with skr_gcrodr_diagnostics */
} skr_config;

enum skr_config_flags { SKR_COLLECT_DIAGNOSTICS = 1 };

/* SolveReport (gmres.py:46-56) minus the vectors. */
typedef struct skr_report {
  int32_t iterations;
  int32_t converged;
  int32_t k_out;          /* recycle columns on exit (0 = empty space) */
  int32_t hist_len;       /* residual_history length */
  int32_t n_checks;       /* restart_checks entries */
  int32_t deflated_steps;
  int32_t warn_bits;      /* reference warnings.warn equivalents, see skr_warn */
  int32_t status_bits;    /* internal dense-kernel status (informational) */
  int32_t zero_rhs;       /* b == 0 early return (gcrodr.py:337-346) */
  int32_t gmres_fallback; /* U stayed None (gcrodr.py:481-483) */
  int32_t cycles;
  int32_t v0_projections; /* cycles whose V_0 was formed from r - C C^T r */
  double true_relative_residual;
  double rnorm;
  double abs_tol;
  double bnorm;
  double device_ms;       /* device time of the solve (CUDA events) */
  double spmv_ortho_bytes;/* algorithmic bytes of the Arnoldi steps */
  double cycle_kernel_ms; /* summed CUDA-event time of the Arnoldi-cycle kernel launches */
  double dense_kernel_ms; /* summed time of the per-cycle recycle-update (dense) launches */
  int32_t launches;       /* kernels this solve launched (incl. speculative no-op cycles) */
  int32_t arnoldi_steps;  /* Arnoldi steps executed (SpMV + ortho), incl. the GMRES cycles */
} skr_report;

enum skr_warn {
  SKR_WARN_SINGULAR_H = 1,
  SKR_WARN_SINGULAR_CROSS = 2,
  SKR_WARN_RANK_DROP = 4,
  SKR_WARN_REFRESH_RANK = 8,
  SKR_WARN_JACOBI_SVD = 16,
};

int skr_version(void);
const char* skr_status_string(int status);
/* number of SMs / L2 bytes of the current device (for reports) */
int skr_device_info(int* sm_count, long long* l2_bytes);

/* y = A x, or y = D^-1 (A x) when apply_prec and A->diag. Bit-exact with
 * scipy's csr_matvec (sequential row sum from 0.0, no FMA) + numpy divide. */
int skr_spmv(const skr_csr* A, const double* x, double* y, int apply_prec, void* stream);
/* r = D^-1 (b - A x) (or b - A x): the reference's explicit residual. */
int skr_residual(const skr_csr* A, const double* b, const double* x, double* r, int apply_prec,
                 void* stream);

/* Stencil form of A (matrix-free 5-/7-point operator; replaces the CSR reads
 * of sparse.py:155-160 csr_matvec on the hot path): the
 * entries of a CSR whose pattern lies on the diagonals {0, +-1, +-sx, +-sxy}
 * with bitwise-symmetric, nonzero off-diagonal values and a diagonal in every
 * row are kept as D, W (-1), S (-sx), B (-sxy): 24 / 32 bytes per row instead
 * of 64 / 88. skr_stencil_build verifies the pattern on the device
 * (stream-ordered, no host sync); a matrix that does not qualify leaves the
 * form disabled and the kernels fall back to the CSR. Returns 0 bytes for
 * invalid offsets (sx >= 2, sxy == 0 or sxy > sx). */
size_t skr_stencil_bytes(int32_t n, int32_t sx, int32_t sxy);
int skr_stencil_build(const skr_csr* A, int32_t sx, int32_t sxy, void* buf, size_t bytes,
                      void* stream);

/* Device assembly of the benchmark configs' FD systems (problems.py assemble;
 * reference problems.py:335-355, :380-383): from the per-cell coefficient
 * field (kind 0: a of -div(a grad u), harmonic-mean faces, wall faces = cell
 * value, negative h^2-scaled diagonal; kind 1: Helmholtz wavenumber k(x),
 * off-diagonals 1, diagonal -2 dim + (k h)^2) on an n^dim interior grid in
 * natural ordering, writes the stencil form (verified flag set; stencil_bytes
 * >= skr_stencil_bytes(n^dim, n, dim == 3 ? n^2 : 0)) and, when values is not
 * NULL, the CSR values in the fixed pattern row_ptr. Bit-identical to the host
 * assembly (same operation order, no FMA contraction). */
int skr_assemble_fd(int32_t kind, int32_t dim, int32_t n, const double* field, double h,
                    const int32_t* row_ptr, double* values, void* stencil, size_t stencil_bytes,
                    void* stream);

/* Device sampling of the configs' coefficient fields (the
 * device counterpart of problems.system_params, which stands in for the
 * reference's samplers kryrec/problems.py:97-162 seeded per system as :488).
 * White noise = Philox4x32-10 (key = (seed_lo, seed_hi ^ cid), counter =
 * (pair_lo, pair_hi, idx, stream)) + Box-Muller; stream 0 of system idx is the
 * field's noise. g = DCT-III_ortho along every axis of xi * coef,
 * coef = 1 / (pi^2 |kappa|^2 + tau^2) (coef_0 = 0), divided by norm; then
 * kind 0: field = g > 0 ? 12 : 3; kind 1: exp(param g); kind 2: param (1 +
 * 0.3 tanh g). dct = [T | T^T], T the n x n orthonormal DCT-III matrix
 * (T[k][j] = c_j cos(pi j (2k + 1) / (2n))). g_out (optional) receives g.
 * Stream-ordered, allocates nothing (work >= skr_grf_workspace_bytes). */
size_t skr_grf_workspace_bytes(int32_t dim, int32_t n);
int skr_grf_sample(int32_t dim, int32_t n, int32_t kind, double tau, double param, double norm,
                   const double* dct, uint64_t seed, uint32_t cid, uint32_t idx, double* field,
                   double* g_out, void* work, size_t work_bytes, void* stream);
/* count N(0,1) samples (times scale) / [0,1) uniforms of (system idx, stream)
 * of the same generator (the C1 right-hand side noise, C2's k0 and centre). */
int skr_philox_normals(int64_t count, uint64_t seed, uint32_t cid, uint32_t idx,
                       uint32_t stream_id, double scale, double* out, void* stream);
int skr_philox_uniforms(int32_t count, uint64_t seed, uint32_t cid, uint32_t idx,
                        uint32_t stream_id, double* out, void* stream);

/* General left preconditioners (kryrec/precond.py:80-145 SOR / ILU(0) / IC(0) /
 * block Jacobi classes, :161-248 the factorizations, :251-312
 * build_preconditioner). skr_precond_build analyses and factors A on the device
 * into buf (>= skr_precond_bytes): dependency levels of the triangular sweeps,
 * the ILU(0) / IC(0) factor on A's own pattern in the reference's operation
 * order (IC(0) on -A when every diagonal entry is negative), M = D / omega + L
 * for SOR, per-block dense LU with partial pivoting (block <= 256) for block
 * Jacobi. A's row_ptr / col_idx (sorted rows) must outlive buf. info (host, may
 * be NULL: then the call does not synchronise) receives [0] = 0 ok, 1 zero (IC:
 * nonpositive) pivot = ZeroPivotError(kind, row = info[1], *value), 2 matrix not
 * symmetric (IC(0) only; ValueError in the reference). skr_precond_apply solves
 * M z = v for ncols columns (in == out allowed); one apply per buffer at a time. */
enum skr_precond_kind { SKR_PC_SOR = 1, SKR_PC_ILU0 = 2, SKR_PC_ICC0 = 3, SKR_PC_BJACOBI = 4 };
size_t skr_precond_bytes(int32_t kind, int32_t n, int32_t nnz, int32_t block);
int skr_precond_build(const skr_csr* A, int32_t kind, double omega, int32_t block, void* buf,
                      size_t bytes, int32_t* info, double* value, void* stream);
int skr_precond_apply(const void* precond, const double* in, double* out, int32_t ncols,
                      int64_t ld_in, int64_t ld_out, void* stream);

size_t skr_gcrodr_workspace_bytes(int32_t n, int32_t m, int32_t k, int32_t max_iter);
/* Solve A x = b with GCRO-DR. U_in (n x k_in, column-major, leading dim ldu)
 * is the previous system's recycle U (its C is not needed: the refresh
 * discards it, gcrodr.py:361-366); U_in may alias the workspace's own U block
 * (chain mode, see skr_gcrodr_recycle_view). x0 may be NULL. x is written.
 * hist/checks (host, may be NULL) receive residual_history and
 * restart_checks (pairs). */
int skr_gcrodr_solve(const skr_csr* A, const double* b, const double* x0, double* x,
                     const skr_config* cfg, const double* U_in, int32_t ldu, int32_t k_in,
                     void* workspace, size_t ws_bytes, skr_report* report, double* hist,
                     int32_t hist_cap, double* checks, int32_t checks_cap, void* stream);
/* The diagnostics the last solve logged with SKR_COLLECT_DIAGNOSTICS
 * (gcrodr.py:372-376, :461-467): up to cap records of 4 doubles (stage: 0 =
 * refresh, 1 = cycle; k; ||op U - C||_F; ||C^T C - I||_F) into out (host).
 * Returns the number of records (>= 0) or a negative status. */
int skr_gcrodr_diagnostics(void* workspace, size_t ws_bytes, int32_t n, int32_t m, int32_t k,
                           int32_t max_iter, double* out, int32_t cap);
/* Device pointers of the recycle pair left in the workspace by the last solve:
 * U (n x k, ld) and C (n x k, ld). */
int skr_gcrodr_recycle_view(void* workspace, size_t ws_bytes, int32_t n, int32_t m, int32_t k,
                            double** U, double** C, int32_t* k_out, int32_t* ld);

/* One linear system of a chain: device CSR, right-hand side, solution out. */
typedef struct skr_system {
  skr_csr A;
  const double* b;
  double* x;
} skr_system;

/* The chain loop (harness.py:233-260) for several independent chains at once,
 * on one GPU: chain c solves systems[chain_first[c] .. chain_first[c+1]) in
 * that order, each solve refreshing from the U its predecessor left in the
 * chain's workspace workspaces[c] (ws_bytes each); one native host thread and
 * CUDA stream per chain, no host round trip between systems. U_first[c]
 * (n x k_first[c], leading dim ldu_first[c]; may be NULL / 0) seeds chain c
 * (e.g. the chain state of a previous call: the workspace's own U block).
 * reports[i] receives system i's report. The chains' cycle kernels use
 * cfg->grid_ctas CTAs each. Returns the first failing status. */
int skr_gcrodr_solve_chains(const skr_system* systems, const int32_t* chain_first,
                            int32_t n_chains, const skr_config* cfg, void* const* workspaces,
                            size_t ws_bytes, const double* const* U_first,
                            const int32_t* ldu_first, const int32_t* k_first,
                            skr_report* reports);

/* Phase clock counters of the last solve (32 x int64: [0,16) dense kernel,
 * csrc/recycle.h SKR_PHASE; [16,24) cycle kernel CTA 0; [30] cycle-kernel
 * grid size, [31] rows per CTA) -- profiling aid. */
int skr_gcrodr_profile(void* workspace, size_t ws_bytes, int32_t n, int32_t m, int32_t k,
                       long long* out32);

/* Greedy nearest-neighbour sort. params: n_sys x P row-major fp64 (device).
 * dist2 fills D2[i - row0][j] = ||p_i - p_j||^2 for i in [row0, row1), all j
 * (binary {v0, v1} batches use an exact bit-count path). chain computes the
 * order from the full D2 (n_sys x n_sys) with the reference's tie-break and a
 * certified argmin: near-ties are re-evaluated in the reference's exact
 * arithmetic (numpy pairwise summation). */
size_t skr_sort_workspace_bytes(int32_t n_sys, int64_t P);
int skr_sort_binary_check(const double* params, int32_t n_sys, int64_t P, double* v0v1,
                          int32_t* is_binary, void* workspace, size_t ws_bytes, void* stream);
int skr_sort_dist2(const double* params, int32_t n_sys, int64_t P, int32_t row0, int32_t row1,
                   int32_t binary, double v0, double v1, double* D2, void* workspace,
                   size_t ws_bytes, void* stream);
int skr_sort_chain(const double* D2, const double* params, int32_t n_sys, int64_t P,
                   int32_t exact_d2, int32_t* order, int32_t* n_certified, void* stream);
/* grouped_sort's bucketing key (sorting.py:96-105: the first principal
 * coordinate of the centered batch, sign rule included) from the full D2
 * matrix: the dominant eigenpair of the double-centered G = -1/2 J D2 J by
 * trace-normalised repeated squaring + power refinement (no SVD). keys:
 * n_sys doubles (device) = sqrt(lambda_1) u_1, the reference's centered @ vt[0]
 * up to rounding. Stream-ordered. */
size_t skr_sort_pca_workspace_bytes(int32_t n_sys);
int skr_sort_pca_keys(const double* D2, const double* params, int32_t n_sys, int64_t P,
                      double* keys, void* workspace, size_t ws_bytes, void* stream);
/* one-call single-GPU greedy_sort (sorting.py:72-80) */
int skr_greedy_sort(const double* params, int32_t n_sys, int64_t P, int32_t* order_host,
                    void* workspace, size_t ws_bytes, void* stream);

/* Single-CTA dense steps on the device (test / diagnostic entry points).
 * H: (m+1) x m column-major (ld), G: (mm+1) x mm, cross: mm x mm. P out:
 * ld_p x cols. ncols points to two int32: ncols[0] = the number of columns
 * (or a negative status), ncols[1] = skr_warn bits (the reference's
 * warnings.warn: singular H -> generalized problem, gcrodr.py:196-199;
 * singular cross-Gram -> pseudoinverse, gcrodr.py:231-235). */
int skr_dense_hr_first(const double* H, int32_t ldh, int32_t m, int32_t k, double* P,
                       int32_t ldp, int32_t* ncols, void* stream);
int skr_dense_hr_next(const double* G, int32_t ldg, const double* cross, int32_t ldx, int32_t mm,
                      int32_t k, double* P, int32_t ldp, int32_t* ncols, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKR_H_ */
