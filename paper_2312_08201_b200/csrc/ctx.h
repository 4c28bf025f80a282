// Internal state of one lyap_ctx (one seed A0).  Not part of the C-ABI.
#pragma once
#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/lyapgpu.h"

namespace lyap {

// Everything that depends on A0 (and Q, E) only: shared by every lyap_ctx made with
// lyap_setup_like from one base (NEXT row f4: several (Bl, Br) configurations for one seed A0).
struct Basis {
  int device = 0;
  double* lam = nullptr;   // npad x 2
  double* Lf = nullptr;    // npad x npad folded Cauchy matrix
  double* Sr = nullptr;    // n x n real eigenvector basis (column-major)
  double* Sinv = nullptr;  // S_r^{-1}
  double* Qr = nullptr;    // S_r^{-1} Q S_r^{-T} (nterms matrices for a v-linear Q)
  double* Er = nullptr;    // S_r^T E S_r
  float* Lf32 = nullptr;   // mixed precision: [hi | lo] float planes of Lf (npad x 2 npad), built on first use
  int lf32_mode = 0;       // split mode Lf32 was built with (1: 3xTF32 hi/lo, 2: one float plane,
                           // 3: 3xFP16 hi/lo half planes of 2^lf_eA Lf in the same buffer)
  int lf_eA = 0;
  ~Basis() {
    cudaSetDevice(device);
    for (double* p : {lam, Lf, Sr, Sinv, Qr, Er})
      if (p) cudaFree(p);
    if (Lf32) cudaFree(Lf32);
  }
};

// Folded seed state that the per-v engine reads.  Folded real coordinates:
// eigen index == coordinate; a conjugate pair occupies coords (2r, 2r+1) = (Re, Im) of the
// representative with Im(lambda) > 0; real eigenvalues follow the pairs, one coord each;
// coords n..npad-1 are zero padding.  Reps: r < npairs are pairs (coord 2r), r >= npairs are real
// (coord r + npairs).
struct Seed {
  int64_t n = 0, k = 0, npad = 0, npairs = 0, nrep = 0;
  double* lam = nullptr;  // npad x 2: eigenvalue (re, im) of the rep owning the coordinate
  double* bhr = nullptr;  // npad x k: folded B^r = S^T Br        [coord][s]
  double* btl = nullptr;  // npad x k: folded B~l = S^{-1} Bl     [coord][t]
  double* F = nullptr;    // nrep x k x k complex (re, im):  T_d block of rep j, F_j[s][t]
  double* Pb = nullptr;   // nrep x 2k x 2k real: diagonal block of the folded T per rep (preconditioner)
  double* g0 = nullptr;   // k x npad folded right-hand side G0 = B^r^T X~0
  double* hf = nullptr;   // k x npad folded trace weights (tau = t0 + 2 <g, hf>)
  double* Lf = nullptr;   // npad x npad folded Cauchy matrix (K1's A operand), row-major
  double* Sr = nullptr;   // n x n real eigenvector basis (column-major), kept for lyap_solution
  double* Qr = nullptr;   // n x n S_r^{-1} Q S_r^{-T} (column-major), kept for lyap_solution
  double t0 = 0.0;
  int nterms = 1;          // right-hand-side terms: Q(v) = sum_i v_i Q_i when qlin (lyap_setup_qlin)
  bool qlin = false;
  double* t0t = nullptr;   // device: t0 of every term
  std::vector<double> t0h; // host copy
  double wcost[LYAP_KMAX] = {};  // ||B~l_t|| ||B^r_t||: weights of the scheduling cost proxy
  double* dwork = nullptr;       // device: [0, k) wcost, [8, 8 + 2k) batch bounding box, [32, ...) log seeds
};

// Batched Krylov engine buffers (slot-major).
struct Engine {
  int b = 0;        // slots of the current run (<= bcap)
  int bcap = 0;     // slots allocated
  int mmax = 0;     // restart length
  int64_t L = 0;    // vector length k * npad
  int64_t ncol = 0; // K1 GEMM columns, b*k*k rounded up to the N tile
  int nchunk = 0;   // chunks of the vector length for the reductions
  int groups = 1;   // slot groups, each on its own stream (K1 of one overlaps the Krylov kernels of the other)
  double *Bop = nullptr, *U = nullptr;            // groups x npad x ncol  (ncol per group)
  float *Bop32 = nullptr, *U32 = nullptr;         // mixed precision: groups x 2 npad x ncol (lo | hi), groups x npad x ncol
  int mp = 0;                                     // mixed-precision mode the buffers were made for
  int* umctr = nullptr;                           // tcgen05 GEMM tile counters (2 per slot group)
  float *xmax = nullptr, *bmax = nullptr;         // 3xFP16: per slot x parameter max |X_t|; per s max |B^r_s|
  float* colscale = nullptr;                      // 3xFP16: per GEMM column unscale factor (groups x ncol)
  double *Xin = nullptr, *X = nullptr;            // b x L
  double *rhs = nullptr, *t0s = nullptr;          // qlin: per-slot G0(v) (b x L) and t0(v) (b)
  double* Qb = nullptr;                           // b x (mmax+1) x L  (unnormalised basis), FP64 engine
  float* Qf = nullptr;                            // the same in FP32 (mixed-precision engine; Qb null)
  float* Minv = nullptr;                          // b x nrep x (2k)^2, FP32 (engine.cuh EngArgs::Minv)
  double *sigma = nullptr, *mask = nullptr;       // b x k
  double *eta = nullptr, *H = nullptr, *cs = nullptr, *sn = nullptr, *e = nullptr, *y = nullptr;
  double *bnorm = nullptr;                        // b
  double *part = nullptr;                         // b x (mmax+2) x nchunk
  double *part3 = nullptr;                        // b x nchunk x 3
  double *part2 = nullptr;                        // b x (mmax+2) x nchunk  (Gram-row partials)
  double *Gq = nullptr;                           // b x (mmax+1)^2 Gram matrix Q^T Q of the basis
  double *cf = nullptr;                           // b x (mmax+1) projection coefficients
  double *Hraw = nullptr;                         // b x (mmax+1) x mmax unrotated Hessenberg (recycle build)
  int *phase = nullptr, *m = nullptr, *vidx = nullptr, *applies = nullptr, *restarts = nullptr;
  // two-level preconditioner (coarse p > 0): flexible basis Zb = P^{-1} q_j, coarse scratch
  double *Zb = nullptr, *Rbuf = nullptr, *Yz = nullptr, *Cc = nullptr, *Wc = nullptr, *Einv = nullptr;
  int pc = 0;                                     // coarse size the buffers were made for
  int* ctrl = nullptr;                            // per group 8 ints: [2]=active slots, [3]=of them VERIFY,
                                                  // [4..5]=applied vectors, [6..7]=of them VERIFY;
                                                  // then 8 shared: [0]=next queue position, [1]=done count
  int* h_ctrl = nullptr;                          // pinned mirror
  int* order = nullptr;                           // queue order (nv_cap)
  int64_t order_cap = 0;
  int* regq = nullptr;                            // queue position -> recycle regime (regq_cap)
  int64_t regq_cap = 0;
  // device-side scheduling scratch (sched.cuh): cost keys, sorted keys, identity indices, CUB temp
  double *skey = nullptr, *skey2 = nullptr;
  int* sidx = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int64_t sched_cap = 0;
};

}  // namespace lyap

// Coarse space of the two-level preconditioner, built on first use.
struct CoarseSpace {
  int p = 0;                       // size (0: off)
  double *Z = nullptr, *TZ = nullptr;     // [Z; T Z]: 2L x p column-major (TZ = Z + L, leading dim 2L)
  double *Phi = nullptr, *Psi = nullptr;  // k x p x p column-major: Z_t^T Z_t, Z_t^T (T Z)_t
  double build_ms = 0.0;
};

// Stability filter tables (stab.cuh), built on first use.
struct StabTables {
  double *wgrid = nullptr, *Gf = nullptr, *Mm = nullptr;
  int F = 0, PR = 0;
  double scale = 1.0, wtail0 = 0.0, rho = 0.0;
};

struct lyap_ctx {
  int device = 0;
  lyap_opts opts{};
  lyap_info info{};
  lyap_stats stats{};
  std::string err;
  cudaStream_t stream = nullptr;  // library-owned stream (used when the caller passes NULL)
  cublasHandle_t cublas = nullptr;
  cusolverDnHandle_t cusolver = nullptr;
  lyap::Seed seed;
  lyap::Engine eng;
  std::shared_ptr<lyap::Basis> basis;  // lam, Lf, Sr, Qr of `seed` point into it
  // recycle spaces (lyap_set_recycle / lyap_build_recycle): nreg x s_rec folded vectors and T U
  int nreg = 0, s_rec = 0;
  double *Ureg = nullptr, *TUreg = nullptr;
  int* sreg = nullptr;  // device: vectors per regime
  std::string reg_seeds;  // nreg x k doubles (log |v| of each regime's seed), host copy
  std::vector<double> auto_box;  // bounding box (lo, hi per parameter) the automatic spaces were built for
  bool recycle_manual = false;   // spaces given by lyap_set_recycle / lyap_build_recycle: no automatic rebuild
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evfork = nullptr, evjoin = nullptr;
  cudaStream_t xstream[4] = {};  // streams of slot groups 1..3 (group 0 runs on `stream`)
  cudaGraphExec_t gexec[4] = {};  // per slot group: the engine iteration graph, kept across calls
  std::vector<cudaEvent_t> prof_evs;  // K1 timing events of the graphs (opts.profile)
  StabTables stab;
  CoarseSpace coarse;
  cublasHandle_t cublas_eng[4] = {};  // per slot group: cuBLAS inside the captured engine iterations
  double* cublas_ws[4] = {};
  double* Spad = nullptr;  // lyap_solution: padded S_r^T and S_r (row-major np x np each)
  cudaEvent_t xjoin[4] = {};
  // mixed precision: per slot group a side stream for the exact (VERIFY) DMMA GEMM, which runs beside
  // the 3xTF32 GEMM of the Krylov steps, and the fork / join events around it
  cudaStream_t mpstream[4] = {};
  // tcgen05 3xTF32 GEMM (umma.cuh): TMA tensor maps of Lf32 and of each slot group's float B operand,
  // rebuilt when the buffers move
  CUtensorMap um_ta{}, um_tb[4]{};
  const void* um_ta_ptr = nullptr;
  const void* um_tb_ptr[4] = {};
  int um_ta_mode = 0, um_tb_mode[4] = {};
  int64_t um_tb_ncol[4] = {};
  cudaEvent_t mpfork[4] = {}, mpjoin[4] = {};
};
