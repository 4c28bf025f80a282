/* lyapgpu.h — C-ABI of the B200 trace(E X(v)) sweep engine (arXiv 2312.08201).
 *
 * The operation (eqs. (Ljap jdba 1), (eq:formA)): for every parameter vector
 * v in R^k of a batch V,
 *
 *     A(v) = A0 - Bl diag(v) Br^T,     A(v) X + X A(v)^T = -Q,     tau(v) = trace(E X(v)).
 *
 * How: lyap_setup factors the seed once, A0 = S Lambda S^{-1} (the complex
 * eigendecomposition of PAPER.md:183, computed on the device from the real LAPACK-style
 * packing), and moves Q, E, Bl, Br into that basis (the offline column of Table 1,
 * PAPER.md:493-506).  lyap_trace_batch then solves, per v, the symmetric nk-dimensional form
 * of the SMW capacitance system eq. (SMW_linearsystem) (reduction in
 * DESIGN.md §2.2) with a batched, right-preconditioned Krylov method on the GPU
 * (preconditioner = the v-dependent exact diagonal blocks of eq. (prec))
 * and returns tau(v) = trace(E X0) + 2 sum G_tj H_jt.
 *
 * Conventions (all calls):
 *   - every matrix is float64, ROW-MAJOR (C order, the same as NumPy / torch);
 *   - host pointers unless a flag says "on device";
 *   - every call returns an lyap_status; on failure lyap_last_error(ctx) (or
 *     lyap_last_error(NULL) when no ctx exists yet) gives a message;
 *   - a ctx is not re-entrant: serialise calls per ctx.  Several ctx per device are fine.
 *   - there is no CPU fallback: with no CUDA device every call returns LYAP_ENODEV.
 */
#ifndef LYAPGPU_H
#define LYAPGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lyap_ctx lyap_ctx; /* opaque; owns all device memory of one seed */

typedef enum {
  LYAP_OK = 0,
  LYAP_EINVAL = 1,     /* bad dims / null pointer / k > LYAP_KMAX / Q not symmetric (rel 1e-13) */
  LYAP_ENOMEM = 2,     /* device allocation failed */
  LYAP_ECUDA = 3,      /* CUDA / cuBLAS / cuSOLVER error */
  LYAP_EEIG = 4,       /* eig(A0) failed, pairing not conjugate, or cond(S) > opts.max_cond_S */
  LYAP_ESINGULAR = 5,  /* min|lambda_i + lambda_j| <= 1e-12 max|lambda|: seed Lyapunov operator
                          singular (the Cauchy matrix needs lambda_i + lambda_j != 0) */
  LYAP_EPARTIAL = 6,   /* trace_batch: some v not converged / non-finite; see status[] */
  LYAP_ENODEV = 7      /* no CUDA device (the library has no CPU path) */
} lyap_status;

/* per-v status codes written to status[i] */
enum { LYAP_V_OK = 0, LYAP_V_NOCONV = 1, LYAP_V_NONFINITE = 2,
       LYAP_V_UNSTABLE = 3 /* opts.check_stable: A(v) has an eigenvalue with Re >= 0; not solved */ };

#define LYAP_KMAX 8

typedef struct {
  double tol;          /* stop when ||g0 - C(v) g|| <= tol ||g0|| (true residual of the nk
                          capacitance system, reading R14). default 1e-12 */
  int32_t max_dim;     /* Krylov restart length m_max; 0 = auto (default) */
  int32_t max_restarts;/* restart cycles before status LYAP_V_NOCONV (default 30) */
  int32_t batch;       /* parameter vectors in flight (slots); 0 = auto (default) */
  int32_t warm_start;  /* 1: a slot starts v from the solution of its previous v; 0 (default):
                          from g = 0 (warm starts were measured to save no iterations, and with
                          them a result would depend on which slot solved which v) */
  double max_cond_S;   /* setup fails with LYAP_EEIG above this 1-norm condition of S (1e8) */
  int32_t device;      /* CUDA device ordinal (default: current device) */
  int32_t profile;     /* 1: time every K1 GEMM launch with CUDA events (lyap_get_stats) */
  int32_t schedule;    /* 1 (default): solve v's in descending order of the cost proxy
                          sum_t |v_t| ||B~l_t|| ||B^r_t|| (largest perturbation first, so the slow
                          systems do not form a tail); 0: in row order of V.  Results are returned
                          in row order either way. */
  int32_t recycle;     /* automatic recycle spaces of size s: -1 (default) and 0 off; > 0 that size.
                          With s > 0, lyap_trace_batch builds the spaces itself (lyap_build_recycle
                          on the 2^k corners of the batch's bounding box, all v > 0) the first time
                          and whenever a batch leaves the box; the build time is in lyap_stats.
                          (Off by default since the pair-block preconditioner: measured c5 909.7 v/s
                          off vs 786.7 with s = 32.) */
  int32_t check_stable;/* 1: the stability filter of PAPER.md:1183 (Example 2: configurations whose
                          A(v) has an eigenvalue with Re >= 0 are discarded) runs first; such v get
                          status LYAP_V_UNSTABLE and trace NaN, are not solved and do NOT make the
                          call return LYAP_EPARTIAL.  See lyap_stable_batch.  default 0 */
  int32_t coarse;      /* size p of the coarse space of the two-level preconditioner:
                          P(v)^{-1} r = y + M(v)^{-1}(r - C(v) y), y = Z E(v)^{-1} Z^T r, E(v) = Z^T C(v) Z,
                          with M(v) the exact pair blocks and Z the p dominant right singular vectors
                          of the off-block coupling T_o (randomized SVD at the first trace_batch).
                          -1 (default) auto: 32 when n k >= 2000, else off; 0 off; > 0 that size
                          (multiple of 8, <= 256).  Recycle spaces are not used together with it. */
  int32_t mixed;       /* mixed-precision iterative refinement: the Krylov steps apply
                          the dense Cauchy part of T with an FP32-accurate tensor-core GEMM (3xFP16 with
                          power-of-two scales, or 3xTF32; operands split hi + lo), every cycle ends once
                          its estimated residual has
                          dropped by mixed_eta, and every cycle starts from the TRUE residual of the
                          exact FP64 operator (DMMA GEMM), so the stopping test (tol, reading R14)
                          is unchanged.  -1 (default) auto: on when n > 1536 (the large-tile
                          K1 configuration, where the T-apply dominates); 0 off; 1 on. */
  double mixed_eta;    /* residual reduction per refinement cycle (default 1e-4) */
} lyap_opts;

typedef struct {
  int64_t n, k;
  int64_t npad;        /* n rounded up to the K1 tile; vectors are k x npad float64 */
  int64_t n_pairs;     /* complex-conjugate eigenpairs of A0 (real eigenvalues: n - 2 n_pairs) */
  double t0;           /* trace(E X0), X0 the seed solution (eq. seedLE) */
  double cond_S;       /* ||S_r||_1 ||S_r^{-1}||_1 of the real eigenvector basis */
  double min_lam_sum;  /* min_{i,j} |lambda_i + lambda_j| */
  double max_abs_lam;
  double setup_ms;     /* device time of lyap_setup */
  int32_t batch, max_dim;
  double wcost[LYAP_KMAX]; /* ||B~l_t|| ||B^r_t||: weights of the scheduling cost proxy
                              sum_t |v_t| wcost[t] (opts.schedule; multi-GPU shard balancing) */
  int32_t coarse;          /* size of the two-level preconditioner's coarse space once built (0: none) */
  double coarse_build_ms;  /* device time of its build (explicit T, randomized SVD, T Z, Gram blocks) */
  int32_t mixed_mode;      /* the Krylov steps' T-apply: 0 FP64 (DMMA); 3 3xFP16 on tcgen05 (npad a multiple
                              of 128; the default under mixed precision); 1 3xTF32 (otherwise, or
                              LYAP_MP_GEMM=tf32x3); 2 a one-plane cuBLAS variant (diagnostics) */
} lyap_info;

typedef struct {
  int64_t k1_launches;     /* K1 (Cauchy-fused T-apply GEMM) launches since the last reset */
  int64_t k1_vectors;      /* parameter-vector columns applied (active slots only) */
  double k1_ms;            /* summed CUDA-event time of the K1 GEMM launches (profile=1) */
  double k1_flops;         /* algorithmic flops of those launches: 2 n^2 k^2 per vector */
  int64_t iterations;      /* engine iterations (one batched T-apply each) */
  int64_t kernel_launches; /* all kernels this library launched */
  double batch_ms;         /* device time of the last lyap_trace_batch */
  double recycle_build_ms; /* time spent building recycle spaces (automatic or lyap_build_recycle) */
  int64_t graph_instantiations; /* engine CUDA graphs instantiated (a repeated call updates them in place) */
  int64_t graph_updates;        /* engine CUDA graphs updated in place (cudaGraphExecUpdate) */
  int64_t k1_exact_vectors;     /* of k1_vectors, those applied with the exact FP64 GEMM (all of them
                                   unless opts.mixed: then the VERIFY applications) */
} lyap_stats;

/* Fills *opts with the defaults above. */
void lyap_default_opts(lyap_opts* opts);

/* Offline stage (Table 1 left column).  Copies every input; the caller may free
 * them on return.  A0: n x n, Bl, Br: n x k, Q: n x n symmetric, E: n x n (symmetrised on input,
 * trace(E X) = trace(((E + E^T)/2) X) since X is symmetric).  opts may be NULL.
 * Errors: LYAP_EINVAL, LYAP_ENOMEM, LYAP_ECUDA, LYAP_EEIG, LYAP_ESINGULAR, LYAP_ENODEV.
 * On success *out owns O(n^2 + n k^2 + batch * m_max * n k) device memory. */
int lyap_setup(int64_t n, int64_t k, const double* A0, const double* Bl, const double* Br,
               const double* Q, const double* E, const lyap_opts* opts, lyap_ctx** out);

/* A right-hand side linear in v (the projected equation eq. (param_projected) of PAPER.md:581-589
 * has Q(v) = -G (I_2 (x) D(v)) G^T = sum_i v_i Q_i): Qk holds k symmetric n x n matrices Q_1..Q_k
 * (k x n x n, row-major) and every v is solved with Q(v) = sum_i v_i Q_i in ONE capacitance system
 * (its right-hand side G0(v) = sum_i v_i G0_i and seed trace t0(v) = sum_i v_i t0_i are linear in v;
 * DESIGN.md §2.7).  Everything else as lyap_setup; lyap_trace_batch*, lyap_solution work unchanged
 * (lyap_setup_like does not take such a base).  Used by the extended-Krylov projection (f1). */
int lyap_setup_qlin(int64_t n, int64_t k, const double* A0, const double* Bl, const double* Br, const double* Qk,
                    const double* E, const lyap_opts* opts, lyap_ctx** out);

/* NEXT row f4: a new context for the same A0, Q, E with other damper / edge
 * configurations (Bl, Br: n x k, k may differ from base's).  Reuses base's eigendecomposition,
 * S_r^{-1}, Q_r, E_r and folded Cauchy matrix (shared, reference-counted: base may be destroyed
 * first); costs two n x n x k DGEMMs plus O(n^2 k^2) instead of the O(n^3) eig.  opts NULL: base's.
 * Errors: LYAP_EINVAL, LYAP_ENOMEM, LYAP_ECUDA. */
int lyap_setup_like(const lyap_ctx* base, int64_t k, const double* Bl, const double* Br, const lyap_opts* opts,
                    lyap_ctx** out);

/* Online stage: traces[i] = trace(E X(V[i,:])) for the nv rows of V (nv x k, row-major).
 * v_on_device = 0: V, traces, status are host pointers; the call is synchronous.
 * v_on_device = 1: all three are device pointers (e.g. torch data_ptr()) and the work is
 *   ordered on cuda_stream (cudaStream_t, NULL = legacy default stream); the call still returns
 *   after the batch completes (the engine polls a device counter).
 * status (nullable): per-v LYAP_V_* codes.  A component v_t == 0 is allowed and means column t
 * is absent ("without loss of generality"); negative v are allowed.
 * Returns LYAP_OK, or LYAP_EPARTIAL if any status[i] != 0 (traces[i] is still the last iterate,
 * NaN if non-finite). */
int lyap_trace_batch(lyap_ctx* ctx, int64_t nv, const double* V, double* traces, int32_t* status,
                     int v_on_device, void* cuda_stream);

/* As lyap_trace_batch, with per-v diagnostics (each nullable, same host/device placement as V):
 * applies[i] = T-applications spent on v (Krylov iterations + verifications),
 * resid[i] = final true relative residual ||g0 - C(v) g|| / ||g0||. */
int lyap_trace_batch_ex(lyap_ctx* ctx, int64_t nv, const double* V, double* traces,
                        int32_t* status, int32_t* applies, double* resid, int v_on_device,
                        void* cuda_stream);

/* NEXT row f4, the stability filter of PAPER.md:1183 (the paper computes the rightmost eigenvalue of
 * A(v) and discards Re >= 0).  nunstable[i] = the number of eigenvalues of A(V[i]) in the open right
 * half-plane, counted with the argument principle on the imaginary axis from the k x k transfer
 * function Br^T (A0 - sI)^{-1} Bl of the seed factors (no eigendecomposition of A(v));
 * -1 when A(v) has an eigenvalue on or numerically at the axis (|det(I - D G(iw))| < 1e-10) or the
 * phase could not be resolved -- treat as unstable.  A(v) is stable iff nunstable[i] == 0.
 * V, nunstable: host pointers (v_on_device = 0, synchronous) or device pointers ordered on cuda_stream. */
int lyap_stable_batch(lyap_ctx* ctx, int64_t nv, const double* V, int32_t* nunstable, int v_on_device,
                      void* cuda_stream);

/* NEXT row f3 (solution recycling between consecutive iterates, PAPER.md:375-377 / 670-671): as
 * lyap_trace_batch_ex with DEVICE pointers only (ordered on cuda_stream), plus
 *   X0   (nullable): nv x (k x npad) folded initial guesses g(v) -- e.g. the solutions of nearby,
 *        previously evaluated v (an optimizer's previous iterates); each v starts from its guess and
 *        is certified by the same true-residual test, so the result does not depend on the guess
 *        beyond the tolerance;
 *   Xout (nullable): nv x (k x npad) the solved folded g(v) of every v (to be passed back as X0). */
int lyap_trace_batch_x(lyap_ctx* ctx, int64_t nv, const double* V, const double* X0, double* Xout, double* traces,
                       int32_t* status, int32_t* applies, double* resid, void* cuda_stream);

int lyap_get_info(const lyap_ctx* ctx, lyap_info* info);
int lyap_get_stats(const lyap_ctx* ctx, lyap_stats* stats);
int lyap_reset_stats(lyap_ctx* ctx);

/* NEXT row f2: the full solution X(v) (n x n, row-major; X is symmetric) for each
 * of the nv rows of V, eq. (Xsmalllastline): the batch is solved as in
 * lyap_trace_batch, then X = S X~ S^T = S_r Y S_r^T with Y = J X~ J^T, X~ = X~0 + L o (B~l G + G^T B~l^T)
 * generated entrywise on the device (the Hadamard product with the Cauchy matrix, never formed as
 * a matrix) for a chunk of v at a time, and the two n^3 products of the whole chunk as two batched
 * FP64 DMMA GEMMs (the engine's k1_dgemm).  Host pointers; X holds nv * n * n doubles; traces
 * (nullable) as in lyap_trace_batch.  O(4 n^3) flops per v. */
int lyap_solution(lyap_ctx* ctx, int64_t nv, const double* V, double* X, double* traces);

/* Recycling across neighbouring v: nreg shared recycle spaces of s folded x-space
 * vectors each (U: HOST, nreg x s x k x npad, the layout of lyap_apply_C) and one seed parameter
 * vector per space (seeds: HOST nreg x k).  T U is computed once here (K1).  In later
 * lyap_trace_batch calls every v is assigned to the space whose seed is nearest in log|v|, and its
 * flexible GMRES uses U as the first s search directions (C(v) u = Delta(v) u - T u costs no T-apply:
 * equivalent to GCRO deflation with span U).  Any U gives the same traces (to the tolerance); a good
 * U (lyap_build_recycle) saves iterations.  nreg = 0 turns recycling off.  Requires s <= m_max - 8. */
int lyap_set_recycle(lyap_ctx* ctx, int32_t nreg, int32_t s, const double* U, const double* seeds);

/* Builds the recycle spaces on the device (GCRO-DR-style selection): for each of
 * the nseeds seed parameter vectors (HOST, nseeds x k, all entries non-zero; e.g. the 2^k corners of
 * the grid) one right-preconditioned GMRES cycle is recorded; the s smallest singular directions of
 * C(v_seed) on its search space Z (the generalised eigenproblem (Hbar^T Hbar) p = theta (Z^T Z) p,
 * cuSOLVER sygvd) give U = Z P, and T U = Delta(v_seed) U - Q Hbar P comes from the Arnoldi relation
 * without any T-apply.  Replaces the current spaces (as lyap_set_recycle).  s <= m_max - 8. */
int lyap_build_recycle(lyap_ctx* ctx, int32_t nseeds, const double* seeds, int32_t s);

/* K1 alone, for kernel tests and the roofline bench: Y = C(sigma) X = sigma o X - T X for nvec
 * folded real vectors (each k x npad, row-major; the layout of DESIGN.md §3).  X, Y, sigma are
 * DEVICE pointers; sigma is nvec x k (NULL: sigma = 0, i.e. Y = -T X).  Ordered on cuda_stream. */
int lyap_apply_C(lyap_ctx* ctx, int64_t nvec, const double* X, const double* sigma, double* Y,
                 void* cuda_stream);

/* As lyap_apply_C, with the dense Cauchy part of T (eqs. (N2M1)/(N1M2)) applied in
 * three reduced-precision passes on the tcgen05 tensor cores (3xFP16 with power-of-two operand scales when
 * npad is a multiple of 128, else 3xTF32; lyap_info.mixed_mode) -- the operator of the mixed-precision
 * Krylov steps; T_d and sigma o X stay FP64.  Relative error ~1e-5 of the Cauchy sums (not an exact apply).
 * Requires mixed precision on for ctx (opts.mixed = 1, or auto with n > 1536): else LYAP_EINVAL. */
int lyap_apply_C_mixed(lyap_ctx* ctx, int64_t nvec, const double* X, const double* sigma, double* Y,
                       void* cuda_stream);

/* Host copies of the folded seed state, for tests (each pointer nullable; sizes from lyap_info):
 *   lam: n x 2 (re, im) eigenvalue per folded coordinate (pair p: coords 2p, 2p+1 both hold the
 *        eigenvalue with positive imaginary part);  bhr, btl: n x k folded  B^r = S^T Br and
 *        B~l = S^{-1} Bl;  F: (n_pairs + n_real) x k x k x 2 complex T_d blocks;
 *   g0, hf: k x npad folded right-hand side and trace weights. */
int lyap_export_state(const lyap_ctx* ctx, double* lam, double* bhr, double* btl, double* F,
                      double* g0, double* hf);

void lyap_destroy(lyap_ctx* ctx);

/* ---- NEXT row f1: extended-Krylov projection (§2.2, Alg. 1) ----------
 * For large n where eig(A0) is unaffordable but solves with A0 are (Assumption 3): one basis of
 * EK_m(A0, P), P = [X0 Br, Bl], for every v; the projected equation eq. (param_projected) is solved by
 * the dense engine above (dimension 4mk; k instances, the right-hand side being linear in v); the
 * space grows by 4k columns per step until the backward error of Prop. 2.1 is
 * <= eps for every v of the batch (Alg. 1; per-v certification).  The result is an APPROXIMATION
 * controlled by eps.
 * lyap_ek_setup: A0 (n x n), Bl, Br (n x k), X0Br = X0 Br (n x k; the seed solution's action, from a
 * closed form or any Lyapunov solver), E (n x n, symmetrised), trEX0 = trace(E X0); all host,
 * row-major.  max_dim caps the basis (default 400 columns).  LU of A0 on the device (cuSOLVER).
 * lyap_ek_trace_batch: host V (nv x k) -> traces (nv); dim_used / bwd_err (nullable): basis size
 * and the largest sampled backward error.  max_steps bounds the expansions of this call.
 * Returns LYAP_OK only when a look-ahead block certified bwd_err <= eps (or the basis reached n
 * columns: the projection is then exact).  LYAP_EPARTIAL (traces still written): the target was not
 * certified -- the basis hit max_dim below n, max_steps ran out, or a projected solve did not
 * converge for some v; bwd_err is then the last certified value (infinity if none). */
typedef struct lyap_ek lyap_ek;
int lyap_ek_setup(int64_t n, int64_t k, const double* A0, const double* Bl, const double* Br, const double* X0Br,
                  const double* E, double trEX0, int32_t max_dim, lyap_ek** out);
int lyap_ek_trace_batch(lyap_ek* ek, int64_t nv, const double* V, double eps, int32_t max_steps, double* traces,
                        int32_t* dim_used, double* bwd_err);
/* As lyap_ek_trace_batch with per-v certification output (Alg. 1): bwd_v[i] = the
 * Prop. 2.1 backward error with which V[i]'s trace was certified (host, nullable), dim_v[i] = the basis
 * size of the space it was taken from (nullable).  Every v is certified separately: its trace comes
 * from the first checked space whose backward error for that v is <= eps. */
int lyap_ek_trace_batch_ex(lyap_ek* ek, int64_t nv, const double* V, double eps, int32_t max_steps, double* traces,
                           double* bwd_v, int32_t* dim_v);
void lyap_ek_destroy(lyap_ek* ek);
const char* lyap_ek_last_error(const lyap_ek* ek);

/* Message of the last failure on this ctx; lyap_last_error(NULL) gives the last failure of the
 * calling thread when no ctx was produced (e.g. a failed lyap_setup).  Never NULL. */
const char* lyap_last_error(const lyap_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* LYAPGPU_H */
