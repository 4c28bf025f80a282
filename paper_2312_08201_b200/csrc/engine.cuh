// Batched right-preconditioned GMRES over parameter vectors.
//
// Each of b "slots" solves one capacitance system C(v) g = g0, C(v) = Delta(v) - T (the symmetric
// nk form of eq. (SMW_linearsystem)), right-preconditioned with the exact
// v-dependent diagonal blocks of C(v) per eigen pair (eq. (prec), p-bar = 0,
// widened by the pair's own Cauchy coupling; see k_pfactor).
// All slots advance in lock step: one batched K1 launch per iteration applies C(v) to every slot's
// current vector.  A slot walks   VERIFY (true residual of its current iterate, trace, convergence)
// -> ITER (Krylov steps, CGS2) -> XUPD (x += P^{-1} Q y) -> VERIFY ...; a converged slot writes
// tau(v) and takes the next v of the batch (device-side queue, deterministic order).  With
// warm_start the new v starts from the previous v's solution in the slot: neighbouring grid points
// recycle each other's solution (the recycling idea of PAPER.md:375-391, in its simplest form).
// Basis vectors are stored unnormalised (q^_i, with eta_i = ||q^_i||): the grid-wide norm is only
// known one kernel later, so the division is folded into the coefficients that use q_i.
#pragma once
#include "common.cuh"
#include "k1.cuh"

namespace lyap {

#ifndef LYAP_RED_CE
#define LYAP_RED_CE 1024
#endif
constexpr int RED_CE = LYAP_RED_CE;  // vector elements per reduction chunk (blocks of k_dots / k_upd)
constexpr int CTRL_RMAX = 16;  // back substitution keeps y in registers: m_max <= 32 * CTRL_RMAX = 512

struct EngArgs {
  int b, mmax, K, nv;
  int64_t L, npad, nrep, npairs, two_np, n;
  int nchunk;
  double tol, tol_inner, t0;
  double eta_rel;  // mixed precision: a cycle also ends once its estimated residual is
                   // eta_rel times the cycle's true starting residual (iterative refinement); 0: off
  int max_restarts, warm;
  const double *V, *g0, *hf, *Pb;  // Pb: per-rep diagonal blocks of T (preconditioner, k_pfactor)
  const int* order;  // queue position -> row of V (null: identity)
  // recycling: nreg shared spaces of s_rec x-space vectors U and their T U; a v
  // whose queue position maps to regime r >= 0 runs flexible GMRES with U_r as its first search
  // directions (C(v) u = Delta(v) u - T u: no T-apply).  regq: queue position -> regime (or -1).
  int s_rec;                 // stride (max size) of a regime space
  const int* sreg;           // per regime: number of vectors (<= s_rec)
  const double *Ureg, *TUreg;
  const int* regq;
  int* su;      // per slot: recycle directions of the current v (0 = none)
  int* reg;     // per slot: regime of the current v
  int record;   // lyap_build_recycle: stop every slot after its first cycle (keep its Krylov data)
  double* Hraw; // unrotated Hessenberg columns (b x (mmax+1) x mmax), written when record != 0
  double *X, *Xin, *Qb, *sigma, *mask, *eta, *H, *e, *y, *bnorm, *part, *part3;
  // mixed precision: the Krylov basis is stored in FP32 (Qf; Qb null) -- a cycle only has to reduce the
  // residual by mixed_eta, and every cycle starts from the exact FP64 residual
  float* Qf;
  // P(v)^{-1} pair blocks, stored in FP32 (an FP32-rounded inverse is still one fixed preconditioner,
  // applied identically by k_prec and the solution update; FP64 arithmetic throughout): half the bytes
  // of the largest per-iteration stream of k_prec
  float* Minv;
  // 3xFP16 T-apply (mixed_mode 3): per slot and parameter max |Xin_t| as float bits (the FP16 column
  // scales of k1_gen16), zeroed by k_pfactor and accumulated by k_prec (atomicMax); null otherwise
  unsigned int* xmaxu;
  double *part2, *Gq, *cf;  // Gram-row partials, Gram matrix Q^T Q of the basis, projection coefficients
  int *phase, *m, *vidx, *applies, *restarts, *ctrl, *newv, *alist;
  int* qctr;      // shared by all slot groups: [0] next queue position, [1] finished v's
  double *cs, *sn;  // Givens rotations (b x mmax each)
  double* traces;
  double* gout;  // optional (lyap_solution, lyap_trace_batch_x): nv x L, the solved folded g of every v
  const double* x0;  // optional (lyap_trace_batch_x): nv x L initial guesses (solution recycling, f3)
  // v-linear right-hand side (lyap_setup_qlin: Q(v) = sum_i v_i Q_i): g0 holds nterms x L terms, t0t
  // nterms seed traces; per slot rhs = sum_i v_i g0_i (b x L) and t0s = sum_i v_i t0_i.  nterms = 0: off
  int nterms;
  const double* t0t;
  double *rhs, *t0s;
  // two-level preconditioner (pc > 0): coarse space Z (L x pc), T Z, Gram blocks
  // Phi_t / Psi_t (k x pc x pc); per slot E(v)^{-1} (pc x pc), flexible basis Zb (as Qb), scratch
  int pc;
  const double *Zc, *Phi, *Psi;  // Zc: [Z; T Z] interleaved, 2L x pc column-major
  double *Einv, *Zb, *Rbuf, *Yz, *Cc, *Wc;  // Yz: per slot [Z w; T Z w] (2L)
  int32_t* status;
  int32_t* out_applies;
  double* out_resid;
};

__device__ __forceinline__ int64_t rep_coord(int64_t rep, int64_t npairs) { return rep < npairs ? 2 * rep : rep + npairs; }

// the basis in its storage type (QT = double: Qb; QT = float: Qf)
template <typename QT>
__device__ __forceinline__ QT* qbase(const EngArgs& a);
template <>
__device__ __forceinline__ double* qbase<double>(const EngArgs& a) { return a.Qb; }
template <>
__device__ __forceinline__ float* qbase<float>(const EngArgs& a) { return a.Qf; }

// ---------------------------------------------------------------- phase advance + v queue
// One block (b <= 1024 threads): XUPD -> VERIFY; FREE slots take the next v's in slot order.
__global__ void k_assign(EngArgs a) {
  __shared__ int wsum[32];
  __shared__ int base_s;
  const int tid = threadIdx.x;
  int flag = 0;
  if (tid < a.b) {
    a.newv[tid] = 0;
    if (a.phase[tid] == PH_XUPD) a.phase[tid] = PH_VERIFY;
    flag = a.phase[tid] == PH_FREE;
  }
  // block exclusive scan of flag
  const int lane = tid & 31, w = tid >> 5;
  int x = flag;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  int off = 0, total = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
    if (i < w) off += wsum[i];
    total += wsum[i];
  }
  // claim `total` consecutive queue positions (the queue is shared by the slot groups)
  if (tid == 0) base_s = total ? atomicAdd(&a.qctr[0], total) : 0;
  __syncthreads();
  const int pos = off + x - flag;
  const int base = base_s;
  if (tid < a.b && flag) {
    const int qpos = base + pos;
    if (qpos < a.nv) {
      const int idx = a.order ? a.order[qpos] : qpos;
      a.vidx[tid] = idx;
      for (int t = 0; t < a.K; ++t) {
        const double v = a.V[(int64_t)idx * a.K + t];
        a.mask[tid * a.K + t] = (v != 0.0) ? 1.0 : 0.0;
        a.sigma[tid * a.K + t] = (v != 0.0) ? 1.0 / v : 0.0;
      }
      a.applies[tid] = 0;
      a.restarts[tid] = 0;
      a.newv[tid] = 1;
      if (a.t0s) {
        double t0 = 0.0;
        for (int t = 0; t < a.nterms; ++t) t0 += a.V[(int64_t)idx * a.K + t] * a.t0t[t];
        a.t0s[tid] = t0;
      }
      // cold start (g = 0): the first residual is the right-hand side itself -- START forms it
      // without a T-apply; a warm start must verify its initial iterate through K1
      a.phase[tid] = (a.warm || a.x0) ? PH_VERIFY : PH_START;
      int r = a.regq ? a.regq[qpos] : -1;
      bool nomask = true;
      for (int t = 0; t < a.K; ++t) nomask = nomask && (a.V[(int64_t)idx * a.K + t] != 0.0);
      if (!nomask || a.s_rec <= 0) r = -1;  // masked rows: C(v) u != Delta u - T u there
      a.reg[tid] = r;
      a.su[tid] = r >= 0 ? a.sreg[r] : 0;
    } else {
      a.phase[tid] = PH_IDLE;
    }
  }
  __syncthreads();
  // active slots after assignment (VERIFY or ITER), compacted for K1: VERIFY slots first (positions
  // [0, nver): with mixed precision they take the exact FP64 apply), then ITER slots, each in slot order.
  // K1-active: VERIFY, and ITER past the recycled directions (those steps need no T-apply)
  int isver = 0, isit = 0;
  if (tid < a.b) {
    const int ph = a.phase[tid];
    isver = ph == PH_VERIFY;
    isit = ph == PH_ITER && a.m[tid] >= a.su[tid];
  }
  int xv = isver, xi = isit;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yv = __shfl_up_sync(0xffffffffu, xv, o), yi = __shfl_up_sync(0xffffffffu, xi, o);
    if (lane >= o) {
      xv += yv;
      xi += yi;
    }
  }
  __shared__ int wsum2[32];
  __syncthreads();
  if (lane == 31) {
    wsum[w] = xv;
    wsum2[w] = xi;
  }
  __syncthreads();
  int offv = 0, offi = 0, nver = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
    if (i < w) {
      offv += wsum[i];
      offi += wsum2[i];
    }
    nver += wsum[i];
  }
  if (isver) a.alist[offv + xv - 1] = tid;
  if (isit) a.alist[nver + offi + xi - 1] = tid;
  const int act = __syncthreads_count(isver || isit);
  if (tid == 0) {
    a.ctrl[2] = act;
    a.ctrl[3] = nver;
    *reinterpret_cast<unsigned long long*>(a.ctrl + 4) += (unsigned long long)act;   // applied vectors
    *reinterpret_cast<unsigned long long*>(a.ctrl + 6) += (unsigned long long)nver;  // of them VERIFY
  }
}

// ---------------------------------------------------------------- preconditioner factor (K2)
// P(v) = the exact diagonal blocks of C(v) = Delta(v) - T in folded real coordinates, one block per
// eigen representative: 2k x 2k for a conjugate pair (the unknowns Re/Im G_tj, t = 1..k), k x k for
// a real eigenvalue.  Pb (setup, k_pblock) holds the block of T: T_d (F_j, eq. (N1M1) / (2,2) block,
// PAPER.md:302-334) PLUS the part of the Cauchy coupling T_o (eqs. (N2M1)/(N1M2))
// that stays inside the pair -- the input index i = conj(j), whose Cauchy entry L_{conj j, j} =
// 1/(2 Re lambda_j) is the largest of its row for light damping.  The paper's eq. (prec)
// (p-bar = 0) keeps only T_d; adding the pair term cuts the Krylov iterations by
// ~40 % at no extra cost per iteration (a 2k x 2k real block costs what a k x k complex one does;
// DESIGN.md §2.4).  Block layout (row, col) = (2s + a, 2t + b), a, b = 0 (Re), 1 (Im); real reps
// use the top-left k x k with the same row stride 2k.  Rows with v_s = 0 are identity rows.
template <int K>
__device__ __forceinline__ constexpr int pb_stride() { return 4 * K * K; }

// Minv[slot][rep] = P(v)_rep^{-1} by in-place Gauss-Jordan with partial pivoting (rows swapped
// during elimination, the matching columns of the inverse swapped back at the end).
// out: element e = r * 2K + c of the inverse at out[(e / 4) * ostride * 4 + e % 4]: Minv is stored in groups
// of four elements, group-major across the reps of a slot, so the threads of a warp -- consecutive reps --
// read and write consecutive float4 (16-byte accesses instead of 64 scalar ones per block at k = 4)
template <int D, int K>
__device__ __forceinline__ void invert_block(const double* __restrict__ pb, const double* mask, const double* sigma,
                                             float* __restrict__ out, int64_t ostride) {
  constexpr int RS = 2 * K, PER = D / K;  // row stride; rows per parameter (2 pair, 1 real)
  double M[D][D];
  int perm[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    const int s = r / PER;
    const double msk = mask[s];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double v = msk != 0.0 ? -pb[r * RS + c] : 0.0;
      if (r == c) v = msk != 0.0 ? v + sigma[s] : 1.0;
      M[r][c] = v;
    }
  }
  for (int c = 0; c < D; ++c) {
    int p = c;
    double best = fabs(M[c][c]);
    for (int r = c + 1; r < D; ++r)
      if (fabs(M[r][c]) > best) {
        best = fabs(M[r][c]);
        p = r;
      }
    perm[c] = p;
    if (p != c)
      for (int j = 0; j < D; ++j) {
        const double t = M[c][j];
        M[c][j] = M[p][j];
        M[p][j] = t;
      }
    const double piv = M[c][c];
    const double inv = piv != 0.0 ? 1.0 / piv : 0.0;  // singular block: zero row (z = 0 there)
    M[c][c] = 1.0;
    for (int j = 0; j < D; ++j) M[c][j] *= inv;
    for (int r = 0; r < D; ++r) {
      if (r == c) continue;
      const double f = M[r][c];
      M[r][c] = 0.0;
      for (int j = 0; j < D; ++j) M[r][j] = fma(-f, M[c][j], M[r][j]);
    }
  }
  for (int c = D - 1; c >= 0; --c) {
    const int p = perm[c];
    if (p != c)
      for (int r = 0; r < D; ++r) {
        const double t = M[r][c];
        M[r][c] = M[r][p];
        M[r][p] = t;
      }
  }
  // elements e = r * 2K + c in groups of four: group g of rep at out[g * ostride * 4 .. + 3] (one 16-byte store)
#pragma unroll
  for (int g = 0; g < ((D - 1) * RS + D - 1) / 4 + 1; ++g) {
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = 4 * g + q, r = e / RS, c = e % RS;
      v[q] = (r < D && c < D) ? (float)M[r < D ? r : 0][c < D ? c : 0] : 0.f;
    }
    *reinterpret_cast<float4*>(out + (int64_t)g * ostride * 4) = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// the Minv block of (slot, rep): element e at minv_of(...)[(e / 4) * nrep * 4 + e % 4]
__device__ __forceinline__ const float* minv_of(const float* Minv, int64_t slot, int64_t rep, int64_t nrep, int S) {
  return Minv + slot * nrep * S + rep * 4;
}

// One thread per (slot with a new v, rep): factor the rep's block; a cold start zeroes X there.
template <int K>
__global__ void __launch_bounds__(128) k_pfactor(EngArgs a) {
  const int slot = blockIdx.y;
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // (k_prec of this iteration accumulates the new maxima; it runs after this kernel on the same stream)
  if (a.xmaxu && blockIdx.x == 0 && threadIdx.x < K) a.xmaxu[slot * K + threadIdx.x] = 0u;
  if (rep >= a.nrep || !a.newv[slot]) return;
  const bool pair = rep < a.npairs;
  float* out = a.Minv + (int64_t)slot * a.nrep * pb_stride<K>() + rep * 4;
  const double* pb = a.Pb + rep * pb_stride<K>();
  if (pair)
    invert_block<2 * K, K>(pb, a.mask + slot * K, a.sigma + slot * K, out, a.nrep);
  else
    invert_block<K, K>(pb, a.mask + slot * K, a.sigma + slot * K, out, a.nrep);
  if (a.rhs) {  // per-slot right-hand side G0(v) = sum_i v_i G0_i at this rep's coordinates
    const int64_t c = rep_coord(rep, a.npairs);
    const int w = pair ? 2 : 1;
    const double* v = a.V + (int64_t)a.vidx[slot] * K;
    for (int t = 0; t < K; ++t)
      for (int q = 0; q < w; ++q) {
        double acc = 0.0;
        for (int i = 0; i < a.nterms; ++i) acc += v[i] * a.g0[(int64_t)i * a.L + t * a.npad + c + q];
        a.rhs[(int64_t)slot * a.L + t * a.npad + c + q] = acc;
      }
  }
  if (a.x0) {  // caller's initial guess for this v (masked rows: column t absent -> 0)
    const int64_t c = rep_coord(rep, a.npairs);
    const int w = pair ? 2 : 1;
    const double* g = a.x0 + (int64_t)a.vidx[slot] * a.L;
    for (int t = 0; t < K; ++t)
      for (int q = 0; q < w; ++q)
        a.X[(int64_t)slot * a.L + t * a.npad + c + q] = a.mask[slot * K + t] != 0.0 ? g[t * a.npad + c + q] : 0.0;
  } else if (!a.warm) {
    const int64_t c = rep_coord(rep, a.npairs);
    const int w = pair ? 2 : 1;
    for (int t = 0; t < K; ++t)
      for (int q = 0; q < w; ++q) a.X[(int64_t)slot * a.L + t * a.npad + c + q] = 0.0;
  }
}

// z = P_rep^{-1} r on the rep's folded coordinates: r[2t + b] (pairs) / r[t] (reals)
template <int K>
__device__ __forceinline__ void apply_pinv(const float* __restrict__ mi, int64_t st, bool pair,
                                           const double (&r)[2 * K], double (&z)[2 * K]) {
  constexpr int RS = 2 * K;
  if (pair) {
    float m[4 * K * K];
#pragma unroll
    for (int g = 0; g < K * K; ++g) {
      const float4 v = *reinterpret_cast<const float4*>(mi + (int64_t)g * st * 4);
      m[4 * g] = v.x, m[4 * g + 1] = v.y, m[4 * g + 2] = v.z, m[4 * g + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < 2 * K; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) acc = fma((double)m[i * RS + j], r[j], acc);
      z[i] = acc;
    }
  } else {
    // real rep: the top-left K x K block (row stride 2K), i.e. the groups up to element (K - 1) * 2K + K - 1
    constexpr int NG = ((K - 1) * RS + K - 1) / 4 + 1;
    float m[4 * NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const float4 v = *reinterpret_cast<const float4*>(mi + (int64_t)g * st * 4);
      m[4 * g] = v.x, m[4 * g + 1] = v.y, m[4 * g + 2] = v.z, m[4 * g + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) acc = fma((double)m[i * RS + j], r[j], acc);
      z[i] = acc;
    }
  }
}

// gather / scatter of a rep's folded coordinates of a k x npad vector (scaled on the way in)
template <int K, typename T>
__device__ __forceinline__ void rep_load(const T* __restrict__ x, int64_t npad, int64_t c, bool pair, double sc,
                                         double (&r)[2 * K]) {
#pragma unroll
  for (int t = 0; t < K; ++t) {
    if (pair) {
      r[2 * t] = sc * (double)x[t * npad + c];
      r[2 * t + 1] = sc * (double)x[t * npad + c + 1];
    } else {
      r[t] = sc * (double)x[t * npad + c];
    }
  }
}
template <int K>
__device__ __forceinline__ void rep_store(double* __restrict__ x, int64_t npad, int64_t c, bool pair,
                                          const double (&z)[2 * K], bool add) {
#pragma unroll
  for (int t = 0; t < K; ++t) {
    if (pair) {
      x[t * npad + c] = add ? x[t * npad + c] + z[2 * t] : z[2 * t];
      x[t * npad + c + 1] = add ? x[t * npad + c + 1] + z[2 * t + 1] : z[2 * t + 1];
    } else {
      x[t * npad + c] = add ? x[t * npad + c] + z[t] : z[t];
    }
  }
}

// 3xFP16: fold this thread's rep values of Xin into the slot's max |Xin_t| (warp max, one atomic per
// warp and t; non-negative floats order like their bit patterns)
template <int K>
__device__ __forceinline__ void note_xmax(const EngArgs& a, int slot, bool pair, const double (&z)[2 * K]) {
  if (!a.xmaxu) return;
  const unsigned mask = __activemask();
  const int leader = __ffs(mask) - 1;
#pragma unroll
  for (int t = 0; t < K; ++t) {
    const double v = pair ? fmax(fabs(z[2 * t]), fabs(z[2 * t + 1])) : fabs(z[t]);
    const unsigned u = __reduce_max_sync(mask, __float_as_uint(__double2float_ru(v)));
    if ((int)(threadIdx.x & 31) == leader) atomicMax(a.xmaxu + slot * K + t, u);
  }
}

// ---------------------------------------------------------------- apply input (K2 apply)
// ITER: Xin = P(v)^{-1} (q^_m / eta_m);  VERIFY: Xin = X.
template <int K, typename QT = double>
__global__ void __launch_bounds__(128) k_prec(EngArgs a) {
  const int slot = blockIdx.y;
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rep >= a.nrep) return;
  const int ph = a.phase[slot];
  if (ph != PH_ITER && ph != PH_VERIFY) return;
  if (ph == PH_ITER && a.m[slot] < a.su[slot]) return;  // recycled direction: no K1 input
  const int64_t c = rep_coord(rep, a.npairs);
  const bool pair = rep < a.npairs;
  double* xin = a.Xin + (int64_t)slot * a.L;
  if (ph == PH_VERIFY) {
    const double* x = a.X + (int64_t)slot * a.L;
    double z[2 * K];
    rep_load<K>(x, a.npad, c, pair, 1.0, z);
    rep_store<K>(xin, a.npad, c, pair, z, false);
    note_xmax<K>(a, slot, pair, z);
    return;
  }
  const int m = a.m[slot];
  const double sc = 1.0 / a.eta[(int64_t)slot * (a.mmax + 1) + m];
  const QT* q = qbase<QT>(a) + ((int64_t)slot * (a.mmax + 1) + m) * a.L;
  double r[2 * K], z[2 * K];
  rep_load<K>(q, a.npad, c, pair, sc, r);
  if (a.pc > 0) {
    // two-level: z = y + M^{-1} (r - C(v) y), y = Z E^{-1} Z^T r and T y (Yz = [Z w; T Z w]) from the coarse GEMMs;
    // C(v) y = sigma o y - T y on unmasked rows, y on masked ones
    double y[2 * K], ty[2 * K];
    rep_load<K>(a.Yz + (int64_t)slot * 2 * a.L, a.npad, c, pair, 1.0, y);       // Z w
    rep_load<K>(a.Yz + (int64_t)slot * 2 * a.L + a.L, a.npad, c, pair, 1.0, ty);  // T Z w
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const double msk = a.mask[slot * K + t], sg = a.sigma[slot * K + t];
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2) {
        const int i = pair ? 2 * t + q2 : t;
        if (!pair && q2) break;
        r[i] -= msk != 0.0 ? sg * y[i] - ty[i] : y[i];
      }
    }
    apply_pinv<K>(minv_of(a.Minv, slot, rep, a.nrep, pb_stride<K>()), a.nrep, pair, r, z);
#pragma unroll
    for (int i = 0; i < 2 * K; ++i) z[i] += y[i];
    rep_store<K>(xin, a.npad, c, pair, z, false);
    rep_store<K>(a.Zb + ((int64_t)slot * (a.mmax + 1) + m) * a.L, a.npad, c, pair, z, false);
    note_xmax<K>(a, slot, pair, z);
    return;
  }
  apply_pinv<K>(minv_of(a.Minv, slot, rep, a.nrep, pb_stride<K>()), a.nrep, pair, r, z);
  rep_store<K>(xin, a.npad, c, pair, z, false);
  note_xmax<K>(a, slot, pair, z);
}

// ---------------------------------------------------------------- two-level preconditioner
// k_cfactor (one CTA per slot with a new v): E(v) = sum_t (v_t != 0 ? sigma_t Phi_t - Psi_t : Phi_t)
// (= Z^T C(v) Z, the Galerkin coarse matrix) and its inverse by Gauss-Jordan with partial pivoting in
// shared memory; Einv[slot] (pc x pc, column-major).
__global__ void __launch_bounds__(256) k_cfactor(EngArgs a, int) {
  extern __shared__ double E[];  // pc x pc column-major, then pc (pivot scratch)
  const int slot = blockIdx.x;
  if (!a.newv[slot]) return;
  const int p = a.pc, tid = threadIdx.x, nt = blockDim.x;
  const int64_t pp = (int64_t)p * p;
  for (int64_t e = tid; e < pp; e += nt) {
    double v = 0.0;
    for (int t = 0; t < a.K; ++t) {
      const double phi = a.Phi[t * pp + e];
      v += a.mask[slot * a.K + t] != 0.0 ? a.sigma[slot * a.K + t] * phi - a.Psi[t * pp + e] : phi;
    }
    E[e] = v;
  }
  __shared__ int piv_s;
  __shared__ double pinv_s;
  int* perm = reinterpret_cast<int*>(E + pp);
  __syncthreads();
  for (int c = 0; c < p; ++c) {
    if (tid < 32) {  // pivot: largest |E(r, c)|, r >= c (first on ties)
      double best = -1.0;
      int arg = c;
      for (int r = c + tid; r < p; r += 32) {
        const double v = fabs(E[(int64_t)c * p + r]);
        if (v > best) {
          best = v;
          arg = r;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oa = __shfl_down_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
          best = ob;
          arg = oa;
        }
      }
      if (tid == 0) {
        piv_s = arg;
        perm[c] = arg;
      }
    }
    __syncthreads();
    const int pr = piv_s;
    if (pr != c)
      for (int j = tid; j < p; j += nt) {
        const double t = E[(int64_t)j * p + c];
        E[(int64_t)j * p + c] = E[(int64_t)j * p + pr];
        E[(int64_t)j * p + pr] = t;
      }
    __syncthreads();
    if (tid == 0) {
      const double pv = E[(int64_t)c * p + c];
      pinv_s = pv != 0.0 ? 1.0 / pv : 0.0;
      E[(int64_t)c * p + c] = 1.0;
    }
    __syncthreads();
    const double inv = pinv_s;
    for (int j = tid; j < p; j += nt) E[(int64_t)j * p + c] *= inv;  // row c
    __syncthreads();
    // eliminate column c from every other row: E(r, j) -= E(r, c) E(c, j); the column-c factors
    // are read before any thread overwrites them (E(r, c) is set to 0 -> the identity column)
    for (int j = tid / 32; j < p; j += nt / 32) {  // warp per column, lanes over rows: coalesced
      if (j == c) continue;
      const double ecj = E[j * p + c];
      for (int r = tid & 31; r < p; r += 32)
        if (r != c) E[j * p + r] = fma(-E[c * p + r], ecj, E[j * p + r]);
    }
    __syncthreads();
    for (int r = tid; r < p; r += nt)
      if (r != c) E[(int64_t)c * p + r] = -E[(int64_t)c * p + r] * E[(int64_t)c * p + c];
    __syncthreads();
  }
  // undo the row swaps as column swaps of the inverse, in reverse order
  for (int c = p - 1; c >= 0; --c) {
    const int pr = perm[c];
    if (pr != c)
      for (int r = tid; r < p; r += nt) {
        const double t = E[(int64_t)c * p + r];
        E[(int64_t)c * p + r] = E[(int64_t)pr * p + r];
        E[(int64_t)pr * p + r] = t;
      }
    __syncthreads();
  }
  double* out = a.Einv + (int64_t)slot * pp;
  for (int64_t e = tid; e < pp; e += nt) out[e] = E[e];
}

// k_cfactor32 (coarse size p <= 32): one WARP per slot with a new v, E(v) held in registers -- lane j
// owns column j (padded with the identity up to 32) -- and inverted by Gauss-Jordan with partial
// pivoting using shuffles only (no shared memory, no barriers).  Same result as k_cfactor.
__global__ void __launch_bounds__(128) k_cfactor32(EngArgs a) {
  __shared__ double Es[4][32 * 33];  // per warp: the 32 x 32 tile, column stride 33 (no bank conflicts)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int slot = blockIdx.x * 4 + w;
  if (slot >= a.b || !a.newv[slot]) return;
  const int p = a.pc, pp = p * p;
  double* T = Es[w];
  double sg[LYAP_KMAX], mk_[LYAP_KMAX];
  for (int t = 0; t < a.K; ++t) {
    sg[t] = a.sigma[slot * a.K + t];
    mk_[t] = a.mask[slot * a.K + t];
  }
  for (int e = lane; e < 32 * 32; e += 32) {  // coalesced assembly of E(v), identity padding
    const int r = e & 31, j = e >> 5;
    double v = (r == j) ? 1.0 : 0.0;
    if (r < p && j < p) {
      v = 0.0;
      for (int t = 0; t < a.K; ++t) {
        const double phi = a.Phi[(int64_t)t * pp + j * p + r];
        v += mk_[t] != 0.0 ? sg[t] * phi - a.Psi[(int64_t)t * pp + j * p + r] : phi;
      }
    }
    T[j * 33 + r] = v;
  }
  __syncwarp();
  double col[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) col[r] = T[lane * 33 + r];
  int perm[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    int pr = c;
    if (lane == c) {  // pivot: largest |E(r, c)|, r >= c (first on ties)
      double best = -1.0;
#pragma unroll
      for (int r = c; r < 32; ++r)
        if (fabs(col[r]) > best) {
          best = fabs(col[r]);
          pr = r;
        }
    }
    pr = __shfl_sync(0xffffffffu, pr, c);
    perm[c] = pr;
    double vpr = 0.0;  // swap rows c and pr in every column
#pragma unroll
    for (int r = c; r < 32; ++r) vpr = (r == pr) ? col[r] : vpr;
#pragma unroll
    for (int r = c + 1; r < 32; ++r) col[r] = (r == pr) ? col[c] : col[r];
    col[c] = vpr;
    const double piv = __shfl_sync(0xffffffffu, col[c], c);
    const double inv = piv != 0.0 ? 1.0 / piv : 0.0;
    if (lane == c) col[c] = 1.0;
    col[c] *= inv;  // row c scaled (E(c, c) = 1 / pivot in lane c)
    const double ecj = col[c];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      if (r == c) continue;
      const double erc = __shfl_sync(0xffffffffu, col[r], c);  // E(r, c) before the update
      if (lane != c) col[r] = fma(-erc, ecj, col[r]);
    }
    if (lane == c) {
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r != c) col[r] = -col[r] * col[c];
    }
  }
#pragma unroll
  for (int c = 31; c >= 0; --c) {  // undo the row swaps as column swaps (lanes c <-> perm[c])
    const int pr = perm[c];
    if (pr != c) {
      const int partner = lane == c ? pr : (lane == pr ? c : lane);
#pragma unroll
      for (int r = 0; r < 32; ++r) col[r] = __shfl_sync(0xffffffffu, col[r], partner);
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) T[lane * 33 + r] = col[r];
  __syncwarp();
  double* out = a.Einv + (int64_t)slot * pp;
  for (int e = lane; e < pp; e += 32) out[e] = T[(e / p) * 33 + e % p];  // coalesced store
}

// k_cpre: Rbuf[slot] = q^_m / eta_m for a slot whose next K1 input is a Krylov direction, else 0
__global__ void __launch_bounds__(256) k_cpre(EngArgs a) {
  const int slot = blockIdx.y;
  const int ph = a.phase[slot];
  const bool on = ph == PH_ITER && a.m[slot] >= a.su[slot];
  double* rb = a.Rbuf + (int64_t)slot * a.L;
  const int m = on ? a.m[slot] : 0;
  const double sc = on ? 1.0 / a.eta[(int64_t)slot * (a.mmax + 1) + m] : 0.0;
  const double* q = a.Qb + ((int64_t)slot * (a.mmax + 1) + m) * a.L;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.L; e += (int64_t)gridDim.x * blockDim.x)
    rb[e] = on ? sc * q[e] : 0.0;
}

// k_cw: Wc[:, slot] = E(v)^{-1} Cc[:, slot]  (one block per slot; rows over threads)
__global__ void __launch_bounds__(128) k_cw(EngArgs a) {
  const int slot = blockIdx.x;
  const int p = a.pc;
  const double* Ei = a.Einv + (int64_t)slot * p * p;
  const double* cc = a.Cc + (int64_t)slot * p;
  for (int r = threadIdx.x; r < p; r += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < p; ++j) acc = fma(Ei[(int64_t)j * p + r], cc[j], acc);
    a.Wc[(int64_t)slot * p + r] = acc;
  }
}

// lyap_build_recycle helpers: Z[:, j] = P(v)^{-1} q^_j / eta_j, or u_j for j < su (the search
// directions of the recorded cycle), and TU = Delta(v) U - C(v) U.
template <int K>
__global__ void __launch_bounds__(128) k_rec_z(EngArgs a, int slot, int m1, double* __restrict__ Z) {
  const int j = blockIdx.y;
  if (j >= m1) return;
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rep >= a.nrep) return;
  const int64_t c = rep_coord(rep, a.npairs);
  const bool pair = rep < a.npairs;
  if (j < a.su[slot]) {  // FGMRES cycle with recycling: the search direction was u_j itself
    const double* u = a.Ureg + ((int64_t)a.reg[slot] * a.s_rec + j) * a.L;
    for (int t = 0; t < K; ++t) {
      Z[(int64_t)j * a.L + t * a.npad + c] = u[t * a.npad + c];
      if (pair) Z[(int64_t)j * a.L + t * a.npad + c + 1] = u[t * a.npad + c + 1];
    }
    return;
  }
  const double sc = 1.0 / a.eta[(int64_t)slot * (a.mmax + 1) + j];
  const double* q = a.Qb + ((int64_t)slot * (a.mmax + 1) + j) * a.L;
  double r[2 * K], z[2 * K];
  rep_load<K>(q, a.npad, c, pair, sc, r);
  apply_pinv<K>(minv_of(a.Minv, slot, rep, a.nrep, pb_stride<K>()), a.nrep, pair, r, z);
  rep_store<K>(Z + (int64_t)j * a.L, a.npad, c, pair, z, false);
}

__global__ void k_rec_tu(const double* __restrict__ U, const double* __restrict__ CU, const double* __restrict__ sig,
                         int64_t L, int64_t npad, int64_t cnt, double* __restrict__ TU) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt * L; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i % L;
    TU[i] = sig[e / npad] * U[i] - CU[i];
  }
}

// ---------------------------------------------------------------- recycled search directions
// ITER step m < su: the search direction is u_m of the slot's regime space and the candidate is
// C(v) u_m = sigma o u_m - (T u)_m, elementwise (the T-apply was paid once, when the space was built).
__global__ void __launch_bounds__(256) k_uapply(EngArgs a) {
  const int slot = blockIdx.y;
  if (a.phase[slot] != PH_ITER) return;
  const int m = a.m[slot];
  if (m >= a.su[slot]) return;
  const int r = a.reg[slot];
  const double* u = a.Ureg + ((int64_t)r * a.s_rec + m) * a.L;
  const double* tu = a.TUreg + ((int64_t)r * a.s_rec + m) * a.L;
  double* w = a.Qb + (int64_t)slot * (a.mmax + 1) * a.L + (int64_t)(m + 1) * a.L;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.L; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e / a.npad);
    w[e] = a.sigma[slot * a.K + t] * u[e] - tu[e];
  }
}

// ---------------------------------------------------------------- orthogonalisation (K3)
// Gram-corrected classical Gram-Schmidt: the new Krylov candidate w is projected with the exact
// projector of the current basis, w' = w - Q G^{-1} Q^T w, G = Q^T Q (normalised basis), i.e. what
// CGS2 approximates with a second pass (G^{-1} ~ 2I - G).  The basis is read twice per iteration
// (one fused dot pass, one update pass) instead of four times; G's new row q_m^T Q comes out of the
// same dot pass and is accumulated in k_gram.
// (Measured on c2 with NumPy: iteration counts identical to CGS2, ||Q^T Q - I|| ~ 1e-14.)
//
// k_dots, ITER: part[slot][i][chunk] = q^_i . w  (i <= m) and part2[slot][i][chunk] = q^_i . q^_m
// (i < m), w = the candidate q^_{m+1} written by K1's epilogue.
// VERIFY: part3[slot][chunk] = (||R||^2, ||rhs||^2, <hf, X>) with R in q^_0.
#ifndef LYAP_DOT_IG
#define LYAP_DOT_IG 64
#endif
constexpr int DOT_IG = LYAP_DOT_IG;  // grid.z of k_dots = min(DOT_Z, ceil((mmax + 1) / DOT_IG)) blocks per chunk
#ifndef LYAP_DOT_Z
#define LYAP_DOT_Z 2
#endif
constexpr int DOT_Z = LYAP_DOT_Z;
template <typename QT = double>
__global__ void __launch_bounds__(256) k_dots(EngArgs a) {
  __shared__ __align__(16) double ws[RED_CE];
  __shared__ double qm[RED_CE];
  __shared__ double red[8];
  const int slot = blockIdx.y, chunk = blockIdx.x;
  const int ph = a.phase[slot];
  const int64_t e0 = (int64_t)chunk * RED_CE;
  const int64_t qs = (int64_t)(a.mmax + 1) * a.L;
  if (ph == PH_VERIFY || ph == PH_START) {
    if (blockIdx.z != 0) return;
    QT* R = qbase<QT>(a) + slot * qs;
    const double* X = a.X + (int64_t)slot * a.L;
    const bool start = ph == PH_START;  // g = 0: R = rhs, written here as q^_0
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int i = threadIdx.x; i < RED_CE; i += blockDim.x) {
      const int64_t e = e0 + i;
      if (e < a.L) {
        const int t = (int)(e / a.npad);
        const double rh = a.mask[slot * a.K + t] * (a.rhs ? a.rhs[(int64_t)slot * a.L + e] : a.g0[e]);
        double r;
        if (start) {
          r = rh;
          R[e] = (QT)rh;
        } else {
          r = R[e];
          s2 += a.hf[e] * X[e];
        }
        s0 += r * r;
        s1 += rh * rh;
      }
    }
    s0 = block_sum(s0, red);
    s1 = block_sum(s1, red);
    s2 = block_sum(s2, red);
    if (threadIdx.x == 0) {
      double* p = a.part3 + ((int64_t)slot * a.nchunk + chunk) * 3;
      p[0] = s0;
      p[1] = s1;
      p[2] = s2;
    }
    return;
  }
  if (ph != PH_ITER) return;
  const int m = a.m[slot];
  // this block's basis vectors: i = 8 (z + Z j) + warp <= m (groups of 8 dealt round-robin over the Z =
  // gridDim.z blocks of a chunk, so short and long cycles both split evenly and a block without work
  // exits before staging; with one block per DOT_IG vectors most blocks of a launch were empty)
  const int i0 = blockIdx.z * 8, istep = 8 * gridDim.z;
  if (i0 > m) return;
  const QT* w = qbase<QT>(a) + slot * qs + (int64_t)(m + 1) * a.L;
  const QT* qlast = qbase<QT>(a) + slot * qs + (int64_t)m * a.L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lim = (int)((a.L - e0) < RED_CE ? (a.L - e0) : RED_CE);
  if constexpr (sizeof(QT) == 4) {
    // FP32 basis: 16-byte loads; w and q_m staged as float4 in shared memory (conflict-free), the products
    // and sums in FP64.  lim is a multiple of 4 (L and the chunk start are).
    float4* ws4 = reinterpret_cast<float4*>(ws);  // RED_CE floats of w, then RED_CE of q_m
    float4* qm4 = ws4 + RED_CE / 4;
    for (int i = threadIdx.x; i < RED_CE / 4; i += blockDim.x) {
      const bool in = 4 * i < lim;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      ws4[i] = in ? reinterpret_cast<const float4*>(w + e0)[i] : z;
      qm4[i] = in ? reinterpret_cast<const float4*>(qlast + e0)[i] : z;
    }
    __syncthreads();
    const int lim4 = lim / 4;
    for (int i = i0 + warp; i <= m; i += istep) {
      const float4* q = reinterpret_cast<const float4*>(qbase<QT>(a) + slot * qs + (int64_t)i * a.L + e0);
      double d0 = 0.0, d1 = 0.0, g0 = 0.0, g1 = 0.0;
      float4 x[RED_CE / 128];
#pragma unroll
      for (int u = 0; u < RED_CE / 128; ++u) {
        const int j = lane + 32 * u;
        x[u] = j < lim4 ? q[j] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < RED_CE / 128; ++u) {
        const int j = lane + 32 * u;
        const float4 wv = ws4[j], qv = qm4[j];
        d0 = fma((double)x[u].x, (double)wv.x, d0);
        d1 = fma((double)x[u].y, (double)wv.y, d1);
        d0 = fma((double)x[u].z, (double)wv.z, d0);
        d1 = fma((double)x[u].w, (double)wv.w, d1);
        g0 = fma((double)x[u].x, (double)qv.x, g0);
        g1 = fma((double)x[u].y, (double)qv.y, g1);
        g0 = fma((double)x[u].z, (double)qv.z, g0);
        g1 = fma((double)x[u].w, (double)qv.w, g1);
      }
      const double d = warp_sum(d0 + d1);
      const double g = warp_sum(g0 + g1);
      if (lane == 0) {
        a.part[((int64_t)slot * (a.mmax + 2) + i) * a.nchunk + chunk] = d;
        if (i < m) a.part2[((int64_t)slot * (a.mmax + 2) + i) * a.nchunk + chunk] = g;
      }
    }
    return;
  }
  for (int i = threadIdx.x; i < RED_CE; i += blockDim.x) {
    const int64_t e = e0 + i;
    ws[i] = e < a.L ? w[e] : 0.0;
    qm[i] = e < a.L ? qlast[e] : 0.0;
  }
  __syncthreads();
  for (int i = i0 + warp; i <= m; i += istep) {
    const QT* q = qbase<QT>(a) + slot * qs + (int64_t)i * a.L + e0;
    double d0 = 0.0, d1 = 0.0, g0 = 0.0, g1 = 0.0;
    int e = lane;
    for (; e + 224 < lim; e += 256) {  // 8 independent loads per lane per round
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = q[e + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        d0 = fma(x[u], ws[e + 32 * u], d0);
        d1 = fma(x[u + 1], ws[e + 32 * u + 32], d1);
        g0 = fma(x[u], qm[e + 32 * u], g0);
        g1 = fma(x[u + 1], qm[e + 32 * u + 32], g1);
      }
    }
    for (; e < lim; e += 32) {
      d0 += q[e] * ws[e];
      g0 += q[e] * qm[e];
    }
    const double d = warp_sum(d0 + d1);
    const double g = warp_sum(g0 + g1);
    if (lane == 0) {
      a.part[((int64_t)slot * (a.mmax + 2) + i) * a.nchunk + chunk] = d;
      if (i < m) a.part2[((int64_t)slot * (a.mmax + 2) + i) * a.nchunk + chunk] = g;
    }
  }
}

// k_gram (one warp per ITER slot): append G's row/column m (G = Q^T Q of the normalised basis,
// G_mm = 1), then c = G^{-1} d to second order: with every new vector projected exactly,
// G = I + E with ||E|| ~ 1e-14, so G^{-1} d = (2I - G) d + O(||E||^2) -- the coefficient CGS2's
// second pass would produce, computed from the Gram row instead of a second sweep over the basis.
// c_i (w.r.t. the normalised q_i) is the Hessenberg column; cf_i = c_i / eta_i multiplies q^_i.
__global__ void __launch_bounds__(256) k_gram(EngArgs a) {
  extern __shared__ double ds[];  // mmax + 1
  const int slot = blockIdx.x;
  if (a.phase[slot] != PH_ITER) return;
  const int ld = a.mmax + 1;
  const int m = a.m[slot];
  const double* eta = a.eta + (int64_t)slot * ld;
  double* G = a.Gq + (int64_t)slot * ld * ld;  // G[i * ld + j], symmetric
  const double* pd = a.part + (int64_t)slot * (a.mmax + 2) * a.nchunk;
  const double* pg = a.part2 + (int64_t)slot * (a.mmax + 2) * a.nchunk;
  for (int i = threadIdx.x; i <= m; i += blockDim.x) {
    double d = 0.0;
    for (int c = 0; c < a.nchunk; ++c) d += pd[(int64_t)i * a.nchunk + c];
    ds[i] = d / eta[i];
    if (i < m) {
      double g = 0.0;
      for (int c = 0; c < a.nchunk; ++c) g += pg[(int64_t)i * a.nchunk + c];
      g /= (eta[i] * eta[m]);
      G[(int64_t)i * ld + m] = g;
      G[(int64_t)m * ld + i] = g;
    } else {
      G[(int64_t)m * ld + m] = 1.0;
    }
  }
  __syncthreads();
  // c = 2 d - G d : one warp per row, the row read coalesced across the lanes
  double* Hc = a.H + (int64_t)slot * ld * a.mmax + (int64_t)m * ld;
  double* cf = a.cf + (int64_t)slot * ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // four rows per warp at a time: 4 independent loads per lane per step of the row sweep
  for (int i = warp * 4; i <= m; i += nw * 4) {
    const double* Gi = G + (int64_t)i * ld;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
    for (int j = lane; j <= m; j += 32) {
      const double dj = ds[j];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u <= m) acc[u] = fma(Gi[(int64_t)u * ld + j], dj, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double sum = warp_sum(acc[u]);
      if (lane == 0 && i + u <= m) {
        const double c = 2.0 * ds[i + u] - sum;
        Hc[i + u] = c;
        cf[i + u] = c / eta[i + u];
        if (a.record) a.Hraw[(int64_t)slot * ld * a.mmax + (int64_t)m * ld + i + u] = c;
      }
    }
  }
}

// k_upd: w' = w - sum_i cf_i q^_i (one read of the basis); part3[slot][chunk][0] = ||w'||^2.
#ifndef LYAP_UPD_UNROLL
#define LYAP_UPD_UNROLL 8
#endif
template <typename QT = double>
__global__ void __launch_bounds__(256) k_upd(EngArgs a) {
  extern __shared__ double cfs[];  // mmax + 1
  __shared__ double red[8];
  const int slot = blockIdx.y, chunk = blockIdx.x;
  if (a.phase[slot] != PH_ITER) return;
  const int m = a.m[slot];
  const int64_t qs = (int64_t)(a.mmax + 1) * a.L;
  for (int i = threadIdx.x; i <= m; i += blockDim.x) cfs[i] = a.cf[(int64_t)slot * (a.mmax + 1) + i];
  __syncthreads();
  QT* w = qbase<QT>(a) + slot * qs + (int64_t)(m + 1) * a.L;
  const QT* Q = qbase<QT>(a) + slot * qs;
  const int64_t e0 = (int64_t)chunk * RED_CE;
  if constexpr (sizeof(QT) == 4) {
    // FP32 basis: each thread owns 4 consecutive elements (one 16-byte load per basis vector)
    static_assert(RED_CE == 4 * 256, "k_upd<float>: one float4 per thread and chunk");
    const int64_t eb = e0 + 4 * threadIdx.x;
    const bool okv = eb < a.L;  // L and e0 are multiples of 4
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int UU = LYAP_UPD_UNROLL;
    int i = 0;
    if (okv) {
      for (; i + UU <= m + 1; i += UU) {
        float4 v[UU];
#pragma unroll
        for (int u = 0; u < UU; ++u) v[u] = *reinterpret_cast<const float4*>(Q + (int64_t)(i + u) * a.L + eb);
#pragma unroll
        for (int u = 0; u < UU; ++u) {
          const double c = cfs[i + u];
          acc[0] = fma(c, (double)v[u].x, acc[0]);
          acc[1] = fma(c, (double)v[u].y, acc[1]);
          acc[2] = fma(c, (double)v[u].z, acc[2]);
          acc[3] = fma(c, (double)v[u].w, acc[3]);
        }
      }
      for (; i <= m; ++i) {
        const double c = cfs[i];
        const float4 v = *reinterpret_cast<const float4*>(Q + (int64_t)i * a.L + eb);
        acc[0] = fma(c, (double)v.x, acc[0]);
        acc[1] = fma(c, (double)v.y, acc[1]);
        acc[2] = fma(c, (double)v.z, acc[2]);
        acc[3] = fma(c, (double)v.w, acc[3]);
      }
    }
    double nrm = 0.0;
    if (okv) {
      float4 wv = *reinterpret_cast<const float4*>(w + eb);
      wv.x = (float)((double)wv.x - acc[0]);
      wv.y = (float)((double)wv.y - acc[1]);
      wv.z = (float)((double)wv.z - acc[2]);
      wv.w = (float)((double)wv.w - acc[3]);
      *reinterpret_cast<float4*>(w + eb) = wv;
      nrm = (double)wv.x * wv.x + (double)wv.y * wv.y + (double)wv.z * wv.z + (double)wv.w * wv.w;
    }
    nrm = block_sum(nrm, red);
    if (threadIdx.x == 0) a.part3[((int64_t)slot * a.nchunk + chunk) * 3] = nrm;
    return;
  }
  // each thread owns 4 elements of the chunk; the basis loop issues 4 independent loads per vector
  constexpr int EPT = RED_CE / 256;
  double acc[EPT];
  bool ok[EPT];
  int64_t eo[EPT];
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    eo[r] = e0 + threadIdx.x + 256 * r;
    ok[r] = eo[r] < a.L;
    acc[r] = 0.0;
  }
  // 8 basis vectors per round: 8 * EPT independent loads in flight per thread (the chain over the
  // basis, not bandwidth, bounds the slot with the longest cycle otherwise)
  constexpr int UU = LYAP_UPD_UNROLL;
  int i = 0;
  for (; i + UU <= m + 1; i += UU) {
    double v[UU][EPT];
#pragma unroll
    for (int u = 0; u < UU; ++u) {
      const QT* q = Q + (int64_t)(i + u) * a.L;
#pragma unroll
      for (int r = 0; r < EPT; ++r) v[u][r] = ok[r] ? (double)q[eo[r]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UU; ++u) {
      const double c = cfs[i + u];
#pragma unroll
      for (int r = 0; r < EPT; ++r) acc[r] = fma(c, v[u][r], acc[r]);
    }
  }
  for (; i <= m; ++i) {
    const double c = cfs[i];
    const QT* q = Q + (int64_t)i * a.L;
#pragma unroll
    for (int r = 0; r < EPT; ++r)
      if (ok[r]) acc[r] = fma(c, (double)q[eo[r]], acc[r]);
  }
  double nrm = 0.0;
#pragma unroll
  for (int r = 0; r < EPT; ++r)
    if (ok[r]) {
      const QT v = (QT)((double)w[eo[r]] - acc[r]);
      w[eo[r]] = v;
      nrm += (double)v * (double)v;  // the norm of the vector as stored
    }
  nrm = block_sum(nrm, red);
  if (threadIdx.x == 0) a.part3[((int64_t)slot * a.nchunk + chunk) * 3] = nrm;
}

// ---------------------------------------------------------------- cycle end: R y = e
// Run by the k_ctrl warp that ends a slot's cycle (no separate launch on the iteration's chain).
// R = the Givens-rotated Hessenberg (m1 x m1 upper triangular, column j at H[j * ld]).  Blocked by
// 32 rows from the bottom: the warp solves a 32 x 32 diagonal block with the block's columns in
// registers (lane l holds row l), so the serial chain is one multiply, one shuffle and one FMA per
// unknown; it then removes the solved unknowns from the rows above (lane l owns rows l + 32 j, a
// coalesced sweep of the block's columns).  e is reduced in place (it is rebuilt at the next cycle).
// (An earlier per-column version spent ~300 cycles per unknown on predicated register selects;
// profiles/r01_backsub_ncu.md.)
__device__ __forceinline__ void warp_backsub(const EngArgs& a, int slot, int lane) {
  const int ld = a.mmax + 1;
  const int m1 = a.m[slot];
  const double* H = a.H + (int64_t)slot * ld * a.mmax;
  double* e = a.e + (int64_t)slot * ld;
  const double* eta = a.eta + (int64_t)slot * ld;
  double* y = a.y + (int64_t)slot * a.mmax;
  const int su = a.su[slot];
  for (int r0 = m1 > 0 ? ((m1 - 1) / 32) * 32 : -1; r0 >= 0; r0 -= 32) {
    const int nb = min(32, m1 - r0);
    const int i = r0 + lane;
    double Rr[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) Rr[c] = (c < nb && lane <= c) ? H[(int64_t)(r0 + c) * ld + i] : 0.0;
    double d = 0.0;
#pragma unroll
    for (int c = 0; c < 32; ++c) d = (c == lane) ? Rr[c] : d;
    const double dinv = d != 0.0 ? 1.0 / d : 0.0;  // a zero pivot (breakdown column) gives y = 0
    double ev = lane < nb ? e[i] : 0.0, yl = 0.0;
#pragma unroll
    for (int c = 31; c >= 0; --c) {
      if (c < nb) {  // warp-uniform
        const double yc = __shfl_sync(0xffffffffu, ev * dinv, c);
        yl = (lane == c) ? yc : yl;
        ev = (lane < c) ? fma(-Rr[c], yc, ev) : ev;
      }
    }
    // u_i raw; P^{-1} q^_i / eta_i (two-level: Zb_i = P^{-1} q^_i / eta_i is stored, coefficient raw)
    if (lane < nb) y[i] = (i < su || a.pc > 0) ? yl : yl / eta[i];
    double yb[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) yb[c] = __shfl_sync(0xffffffffu, yl, c);
    for (int r = lane; r < r0; r += 32) {  // r0 is a multiple of 32: uniform trip count
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        if (c < nb) acc0 = fma(H[(int64_t)(r0 + c) * ld + r], yb[c], acc0);
        if (c + 1 < nb) acc1 = fma(H[(int64_t)(r0 + c + 1) * ld + r], yb[c + 1], acc1);
      }
      e[r] -= acc0 + acc1;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- per-slot control (K4)
// one warp per slot: VERIFY -> done / restart;  ITER -> Hessenberg column, Givens, cycle end.
__global__ void __launch_bounds__(128) k_ctrl(EngArgs a) {
  const int slot = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (slot >= a.b) return;
  const int ph = a.phase[slot];
  const int ld = a.mmax + 1;
  double* H = a.H + (int64_t)slot * ld * a.mmax;
  double* e = a.e + (int64_t)slot * ld;
  double* eta = a.eta + (int64_t)slot * ld;
  double* cs = a.cs + (int64_t)slot * a.mmax;
  double* sn = a.sn + (int64_t)slot * a.mmax;
  const double* p3 = a.part3 + (int64_t)slot * a.nchunk * 3;
  if (ph == PH_VERIFY || ph == PH_START) {
    if (lane != 0) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int c = 0; c < a.nchunk; ++c) {
      s0 += p3[c * 3];
      s1 += p3[c * 3 + 1];
      s2 += p3[c * 3 + 2];
    }
    const double rho = sqrt(s0), bn = sqrt(s1), tr = (a.t0s ? a.t0s[slot] : a.t0) + 2.0 * s2;
    const int ap = (ph == PH_VERIFY) ? ++a.applies[slot] : a.applies[slot];  // START needs no T-apply
    const bool bad = !isfinite(rho) || !isfinite(tr);
    const bool conv = rho <= a.tol * bn;
    if (bad || conv || a.restarts[slot] >= a.max_restarts) {
      const int idx = a.vidx[slot];
      a.traces[idx] = bad ? __longlong_as_double(0x7ff8000000000000LL) : tr;
      if (a.status) a.status[idx] = bad ? LYAP_V_NONFINITE : (conv ? LYAP_V_OK : LYAP_V_NOCONV);
      if (a.out_applies) a.out_applies[idx] = ap;
      if (a.out_resid) a.out_resid[idx] = bn > 0.0 ? rho / bn : rho;
      a.phase[slot] = PH_FREE;
      atomicAdd(&a.qctr[1], 1);
    } else {
      // safety net: a v whose recycled space has not helped within two cycles runs plain GMRES
      if (a.restarts[slot] >= 2) a.su[slot] = 0;
      eta[0] = rho;
      e[0] = rho;
      a.m[slot] = 0;
      a.bnorm[slot] = bn;
      a.phase[slot] = PH_ITER;
    }
    return;
  }
  if (ph != PH_ITER) return;
  // the sequential Givens chain runs on a shared-memory copy of the column (one coalesced load)
  extern __shared__ double sm_ctrl[];
  const int wslot = threadIdx.x >> 5;
  double* hs = sm_ctrl + (int64_t)wslot * 4 * (a.mmax + 2);  // column m of H (m + 2 entries)
  double* css = hs + (a.mmax + 2);
  double* sns = css + (a.mmax + 2);
  double* ys = sns + (a.mmax + 2);
  const int m = a.m[slot];
  double* Hc = H + (int64_t)m * ld;
  for (int i = lane; i <= m; i += 32) hs[i] = Hc[i];
  for (int i = lane; i < m; i += 32) {
    css[i] = cs[i];
    sns[i] = sn[i];
  }
  __syncwarp();
  int done = 0;
  if (lane == 0) {
    double s = 0.0;
    for (int c = 0; c < a.nchunk; ++c) s += p3[c * 3];
    const double hn = sqrt(s);
    a.applies[slot] += 1;
    eta[m + 1] = hn > 0.0 ? hn : 1.0;
    if (a.record) a.Hraw[(int64_t)slot * ld * a.mmax + (int64_t)m * ld + m + 1] = hn;
    double hi = hs[0];
    for (int i = 0; i < m; ++i) {  // apply the previous rotations to the new column
      const double hi1 = hs[i + 1];
      hs[i] = css[i] * hi + sns[i] * hi1;
      hi = -sns[i] * hi + css[i] * hi1;
    }
    const double x1 = hi, x2 = hn;
    const double r = hypot(x1, x2);
    const double c = r > 0.0 ? x1 / r : 1.0, sv = r > 0.0 ? x2 / r : 0.0;
    cs[m] = c;
    sn[m] = sv;
    hs[m] = r;
    hs[m + 1] = 0.0;
    e[m + 1] = -sv * e[m];
    e[m] = c * e[m];
    const double est = fabs(e[m + 1]);
    const bool breakdown = !(hn > 1e-300 * a.bnorm[slot]);
    done = (est <= fmax(a.tol_inner * a.bnorm[slot], a.eta_rel * eta[0])) || (m + 1 >= a.mmax) || breakdown ||
           !isfinite(est);
    // a recycled direction dependent on the current space is not a "lucky" breakdown: finish the
    // cycle and run this v's restarts as plain GMRES
    // (su itself must stay until this cycle's update: its first su search directions are u_i;
    // counting the cycle twice makes the safety net below drop the space at the next restart)
    if (breakdown && m < a.su[slot]) a.restarts[slot] = max(a.restarts[slot], 1);
    a.m[slot] = m + 1;
  }
  __syncwarp();
  for (int i = lane; i <= m + 1; i += 32) Hc[i] = hs[i];
  done = __shfl_sync(0xffffffffu, done, 0);
  if (!done) return;
  if (lane == 0) {
    a.restarts[slot] += 1;
    if (a.record) {  // keep q^_0..q^_m1, H, eta, Minv of this cycle for the recycle-space build
      a.phase[slot] = PH_IDLE;
      atomicAdd(&a.qctr[1], 1);
    } else {
      a.phase[slot] = PH_XUPD;
    }
  }
  if (!a.record) {
    __syncwarp();  // the rotated column (Hc) and e[m], e[m + 1] are visible to the whole warp
    warp_backsub(a, slot, lane);
  }
}

// k_gout (lyap_solution only): a slot that finished its v in this iteration's k_ctrl is FREE until
// the next k_assign; copy its solution g to gout[vidx].
__global__ void __launch_bounds__(256) k_gout(EngArgs a) {
  const int slot = blockIdx.y;
  if (a.phase[slot] != PH_FREE) return;
  const int64_t idx = a.vidx[slot];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.L; e += (int64_t)gridDim.x * blockDim.x)
    a.gout[idx * a.L + e] = a.X[(int64_t)slot * a.L + e];
}


// ---------------------------------------------------------------- solution update
// XUPD: X += U y_U + P(v)^{-1} (sum_{i>=su} y_i q^_i)   (y already carries the 1/eta_i).  One kernel:
// a block owns a window of 64 coordinates for all k rows (pairs never straddle it: the window starts
// at an even coordinate), forms the basis combination there (64 elements x 4 slices of the basis
// index, reduced in shared memory), then applies the k x k P^{-1} block of every representative in
// the window.
template <int K, typename QT = double>
__global__ void __launch_bounds__(256) k_xcomb(EngArgs a) {
  // window of W coordinates; FP32 basis: 128 coordinates as 32 float4 columns x 8 slices of the basis index
  // (16-byte loads), FP64 basis: 64 coordinates x 4 slices
  constexpr bool F4 = sizeof(QT) == 4;
  constexpr int W = F4 ? 128 : 64, NS = F4 ? 8 : 4;
  __shared__ double ys[1024];
  __shared__ double red[NS][W];
  __shared__ double xs[K][W];
  const int slot = blockIdx.y;
  if (a.phase[slot] != PH_XUPD) return;
  const int m1 = a.m[slot];
  const int su = min(a.su[slot], m1);
  const double* ysl = a.y + (int64_t)slot * a.mmax;
  for (int i = threadIdx.x; i < m1; i += blockDim.x) ys[i] = i < su ? 0.0 : ysl[i];
  __syncthreads();
  const QT* Qb0 = qbase<QT>(a);
  if constexpr (sizeof(QT) == 8)
    if (a.pc > 0) Qb0 = (const QT*)a.Zb;  // two-level: Z_j = P^{-1} q_j (FP64 basis only)
  const QT* Q = Qb0 + (int64_t)slot * (a.mmax + 1) * a.L;
  double* X = a.X + (int64_t)slot * a.L;
  const int el = F4 ? (threadIdx.x & 31) : (threadIdx.x & 63), sl = F4 ? (threadIdx.x >> 5) : (threadIdx.x >> 6);
  for (int64_t c0 = (int64_t)blockIdx.x * W; c0 < a.npad; c0 += (int64_t)gridDim.x * W) {
    if constexpr (F4) {
      const int64_t c = c0 + 4 * el;  // npad is a multiple of 64: a float4 column is inside or outside as a whole
#pragma unroll 1
      for (int t = 0; t < K; ++t) {
        const int64_t e = (int64_t)t * a.npad + c;
        double s[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u][0] = s[u][1] = s[u][2] = s[u][3] = 0.0;
        if (c < a.npad) {
          int i = sl;
          for (; i + 3 * NS < m1; i += 4 * NS) {  // 4 independent 16-byte basis loads per step
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4*>(Q + (int64_t)(i + u * NS) * a.L + e);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double y = ys[i + u * NS];
              s[u][0] = fma(y, (double)v[u].x, s[u][0]);
              s[u][1] = fma(y, (double)v[u].y, s[u][1]);
              s[u][2] = fma(y, (double)v[u].z, s[u][2]);
              s[u][3] = fma(y, (double)v[u].w, s[u][3]);
            }
          }
          for (; i < m1; i += NS) {
            const float4 v = *reinterpret_cast<const float4*>(Q + (int64_t)i * a.L + e);
            const double y = ys[i];
            s[0][0] = fma(y, (double)v.x, s[0][0]);
            s[0][1] = fma(y, (double)v.y, s[0][1]);
            s[0][2] = fma(y, (double)v.z, s[0][2]);
            s[0][3] = fma(y, (double)v.w, s[0][3]);
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) red[sl][4 * el + r] = (s[0][r] + s[2][r]) + (s[1][r] + s[3][r]);
        __syncthreads();
        if (threadIdx.x < W) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < NS; ++q) acc += red[q][threadIdx.x];
          xs[t][threadIdx.x] = acc;
        }
        __syncthreads();
      }
    } else {
      const int64_t c = c0 + el;
#pragma unroll 1
      for (int t = 0; t < K; ++t) {
        const int64_t e = (int64_t)t * a.npad + c;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (c < a.npad) {
          int i = sl;
          for (; i + 12 < m1; i += 16) {  // 4 independent basis loads per step
            s0 = fma(ys[i], (double)Q[(int64_t)i * a.L + e], s0);
            s1 = fma(ys[i + 4], (double)Q[(int64_t)(i + 4) * a.L + e], s1);
            s2 = fma(ys[i + 8], (double)Q[(int64_t)(i + 8) * a.L + e], s2);
            s3 = fma(ys[i + 12], (double)Q[(int64_t)(i + 12) * a.L + e], s3);
          }
          for (; i < m1; i += 4) s0 = fma(ys[i], (double)Q[(int64_t)i * a.L + e], s0);
        }
        red[sl][el] = (s0 + s2) + (s1 + s3);
        __syncthreads();
        if (sl == 0) xs[t][el] = (red[0][el] + red[1][el]) + (red[2][el] + red[3][el]);
        __syncthreads();
      }
    }
    if (su > 0) {  // recycled directions enter x directly (not through P^{-1})
      const double* U = a.Ureg + (int64_t)a.reg[slot] * a.s_rec * a.L;
      for (int idx = threadIdx.x; idx < K * W; idx += blockDim.x) {
        const int64_t cc = c0 + (idx % W);
        if (cc >= a.npad) continue;
        const int64_t e = (int64_t)(idx / W) * a.npad + cc;
        double acc = 0.0;
        for (int i = 0; i < su; ++i) acc = fma(ysl[i], U[(int64_t)i * a.L + e], acc);
        X[e] += acc;
      }
      __syncthreads();
    }
    if (a.pc > 0) {  // flexible basis: the directions are already preconditioned
      for (int idx = threadIdx.x; idx < K * W; idx += blockDim.x) {
        const int64_t cc = c0 + (idx % W);
        if (cc < a.npad) X[(int64_t)(idx / W) * a.npad + cc] += xs[idx / W][idx % W];
      }
      __syncthreads();
      continue;
    }
    if (threadIdx.x < W) {
      const int64_t cc = c0 + threadIdx.x;
      const bool pair = cc < 2 * a.npairs;
      const int64_t rep = pair ? cc / 2 : cc - a.npairs;
      if (!(pair && (cc & 1)) && rep < a.nrep) {
        double r[2 * K], z[2 * K];
#pragma unroll
        for (int t = 0; t < K; ++t) {
          if (pair) {
            r[2 * t] = xs[t][threadIdx.x];
            r[2 * t + 1] = xs[t][threadIdx.x + 1];
          } else {
            r[t] = xs[t][threadIdx.x];
          }
        }
        apply_pinv<K>(minv_of(a.Minv, slot, rep, a.nrep, pb_stride<K>()), a.nrep, pair, r, z);
        rep_store<K>(X, a.npad, cc, pair, z, true);
      }
    }
    __syncthreads();
  }
}

}  // namespace lyap

